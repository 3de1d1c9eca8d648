"""Quick first-light check on the GPU box: swap bytes + per-model parity vs the oracle."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import synth, oracle
from paper_2306_03622_b200 import Runtime

names = sys.argv[1:] or ["mlp-small", "mlp", "bert-tiny", "gpt2-tiny", "resnet-tiny"]
rt = Runtime(pool_bytes=8 << 30)
for n in names:
    spec = synth.build_model(n)
    w = spec.build_weights()
    x = spec.make_input()
    mid = rt.register_spec(spec, w)
    t = time.time()
    try:
        r = rt.invoke(mid, x)
    except Exception as e:
        print(n, "INVOKE FAILED", e, flush=True)
        continue
    res = rt.read_resident(mid)
    store = rt.read_store(mid)
    same = np.array_equal(res, store)
    ref = oracle.output(spec, w, x).reshape(-1)
    got = r.output.astype(np.float64).reshape(-1)
    err = np.max(np.abs(got - ref)) / max(1e-30, np.max(np.abs(ref)))
    r2 = rt.invoke(mid, x)
    print(f"{n}: bytes_exact={same} rel_err={err:.3e} warm_equal={np.array_equal(r2.output, r.output)} "
          f"cold={r.stats['device_ms']:.3f}ms swap={r.stats['swap_ms']:.3f}ms {r.stats['link_gbps']:.1f}GB/s "
          f"warm={r2.stats['device_ms']:.3f}ms", flush=True)
rt.close()
