# k_gemm2 in the invoke graph: resident BERT-base / GPT-2-2L by target pair count (token tile), vs k_gemm.
cd $GRAFT_REPO_ROOT
for v in "X=1" "FSW_GEMM_2CTA=1 FSW_GEMM_2CTA_PAIRS=20" "FSW_GEMM_2CTA=1 FSW_GEMM_2CTA_PAIRS=40" "FSW_GEMM_2CTA=1 FSW_GEMM_2CTA_PAIRS=74" "FSW_GEMM_2CTA=1 FSW_GEMM_2CTA_PAIRS=150"; do
env $v timeout 300 python - <<'PY'
import os, sys, numpy as np; sys.path.insert(0, ".")
import synth
from paper_2306_03622_b200 import Runtime
with Runtime(gpu_ids=[0], pool_bytes=16 << 30) as rt:
    out = []
    for name in ("bert-base", "gpt2-2L"):
        spec = synth.build_model(name); mid = rt.register_spec(spec, spec.build_weights()); x = spec.make_input()
        rt.invoke(mid, x, gpu=0)
        d = [rt.invoke(mid, x, gpu=0).stats["device_ms"] for _ in range(30)]
        out.append(f"{name} resident {np.median(d[5:]):.4f}")
    print(os.environ.get("FSW_GEMM_2CTA", "k_gemm"), "pairs", os.environ.get("FSW_GEMM_2CTA_PAIRS", "-"), *out, flush=True)
PY
done
