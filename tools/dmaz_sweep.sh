cd $GRAFT_REPO_ROOT
for taper in 0.25 0.5 0.75; do for ramp in 0 4; do
  FSW_DMAZ_TAPER=$taper FSW_DMAZ_RAMP=$ramp timeout 300 python - <<PY 2>&1 | tail -9
import sys, numpy as np; sys.path.insert(0, ".")
import synth
from paper_2306_03622_b200 import ENGINE_DMAZ, Runtime
with Runtime(gpu_ids=[0], pool_bytes=16 << 30) as rt:
    for name in ("resnet50", "bert-base", "gpt2-xl"):
        spec = synth.build_model(name); mid = rt.register_spec(spec, spec.build_weights(), link_code=True); x = spec.make_input()
        for grp in (64 << 20, 128 << 20, 256 << 20):
            d = []
            for i in range(14 if name != "gpt2-xl" else 6):
                rt.evict(mid); st = rt.invoke(mid, x, gpu=0, engine=ENGINE_DMAZ, dma_group_bytes=grp).stats; d.append(st["device_ms"])
            print(f"taper=$taper ramp=$ramp {name:9s} grp={grp>>20:3d}M p50 {np.median(d[3:]):.4f} copies {st['n_copies']}", flush=True)
        rt.unregister(mid)
PY
done; done
