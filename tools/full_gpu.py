"""Full-size parity + cold/warm timing + swap-kernel sweep on the GPU box (exploration tool)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import synth, oracle
from paper_2306_03622_b200 import Runtime, NO_OVERLAP, DMA_BASELINE

names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["bert-base", "resnet50", "gpt2-2L"]
sweep = "--sweep" in sys.argv
rt = Runtime(pool_bytes=40 << 30)
for n in names:
    t0 = time.time()
    spec = synth.build_model(n)
    w = spec.build_weights()
    x = spec.make_input()
    t1 = time.time()
    mid = rt.register_spec(spec, w)
    t2 = time.time()
    info = rt.model_info(mid)
    r = rt.invoke(mid, x)
    same = np.array_equal(rt.read_resident(mid), rt.read_store(mid))
    t3 = time.time()
    ref = oracle.output(spec, w, x).reshape(-1)
    t4 = time.time()
    got = r.output.astype(np.float64).reshape(-1)
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    print(f"{n}: store={info['store_bytes']} gen={t1-t0:.1f}s reg={t2-t1:.1f}s oracle={t4-t3:.1f}s bytes_exact={same} rel_err={err:.3e}", flush=True)
    def cold(**kw):
        rt.evict(mid)
        return rt.invoke(mid, x, **kw).stats
    for mode, kw in [("default", {}), ("no_overlap", {"flags": NO_OVERLAP}), ("dma", {"flags": DMA_BASELINE})]:
        st = [cold(**kw) for _ in range(8)][3:]
        d = np.median([s["device_ms"] for s in st]); sw = np.median([s["swap_ms"] for s in st])
        tail = np.median([s["compute_tail_ms"] for s in st]); tot = np.median([s["total_ms"] for s in st])
        print(f"   cold[{mode}]: device={d:.3f}ms total={tot:.3f}ms swap={sw:.3f}ms ({info['store_bytes']/sw/1e6:.1f} GB/s) tail={tail:.3f}ms", flush=True)
    wm = [rt.invoke(mid, x).stats for _ in range(10)][3:]
    print(f"   warm: device={np.median([s['device_ms'] for s in wm]):.3f}ms total={np.median([s['total_ms'] for s in wm]):.3f}ms", flush=True)
    if sweep:
        for ctas in [8, 16, 32, 64, 128]:
            for chunk in [64 << 10, 256 << 10, 1 << 20]:
                st = [cold(copy_ctas=ctas, chunk_bytes=chunk) for _ in range(5)][2:]
                sw = np.median([s["swap_ms"] for s in st]); d = np.median([s["device_ms"] for s in st])
                print(f"   sweep ctas={ctas:4d} chunk={chunk>>10:5d}K: device={d:.3f} swap={sw:.3f}ms {info['store_bytes']/sw/1e6:.1f} GB/s", flush=True)
    rt.unregister(mid)
rt.close()
