cd $GRAFT_REPO_ROOT
for v in "FSW_GEMM_2CTA=1" "X=1"; do
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g2_launch_$v.csv python tools/profile_target.py bert-base 1 > /dev/null 2>&1
  echo "== $v"; python tools/ncu_summary.py gpurun_out/g2_launch_$v.csv | head -8
done
# PDL off for GEMMs (mask without the GEMM bit) and on, resident BERT
for m in "" "FSW_PDL_MASK=0"; do env $m timeout 300 python - <<'PY'
import os, sys, numpy as np; sys.path.insert(0, ".")
import synth
from paper_2306_03622_b200 import Runtime
with Runtime(gpu_ids=[0], pool_bytes=8 << 30) as rt:
    spec = synth.build_model("bert-base"); mid = rt.register_spec(spec, spec.build_weights()); x = spec.make_input()
    rt.invoke(mid, x, gpu=0)
    for env2 in ["2cta"]:
        d = [rt.invoke(mid, x, gpu=0).stats["device_ms"] for _ in range(30)]
        print("PDL_MASK", os.environ.get("FSW_PDL_MASK", "default"), "resident", np.median(d[5:]))
PY
done
