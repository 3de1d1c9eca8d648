# DMAZ copy-group schedule for format v4 (BERT-base): tail taper x head ramp x group cap, 30 timed cold
# invokes after 15 untimed ones per point (env hooks are read once per process: one process per pair).
cd $GRAFT_REPO_ROOT
python -m paper_2306_03622_b200.build >/dev/null
for taper in 0.35 0.5 0.65; do for ramp in 0 2 4; do
  FSW_DMAZ_TAPER=$taper FSW_DMAZ_RAMP=$ramp timeout 300 python - <<PY 2>&1 | tail -3
import sys, numpy as np; sys.path.insert(0, ".")
import synth
from paper_2306_03622_b200 import ENGINE_DMAZ, Runtime
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    spec = synth.build_model("bert-base"); mid = rt.register_spec(spec, spec.build_weights(), link_code=True); x = spec.make_input()
    for grp in (32 << 20, 64 << 20, 128 << 20):
        d = []
        for i in range(45):
            rt.evict(mid); st = rt.invoke(mid, x, gpu=0, engine=ENGINE_DMAZ, dma_group_bytes=grp).stats; d.append(st["device_ms"])
        print(f"taper=$taper ramp=$ramp grp={grp>>20:3d}M p50 {np.median(d[15:]):.4f} copies {st['n_copies']}", flush=True)
PY
done; done
