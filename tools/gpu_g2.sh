# 2-CTA GEMM inside libfsw: GPU parity / invariance / edge suites, then resident and cold timings vs the 1-CTA path.
cd $GRAFT_REPO_ROOT
python -m paper_2306_03622_b200.build >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invariance.py tests/test_gpu_edges.py -x -q 2>&1 | tail -4
for v in "FSW_GEMM_2CTA=1" "X=1"; do
  echo "== ${v:-2cta}"
  env $v timeout 600 python tools/linkcode_bench.py bert-base gpt2-xl --reps 10 2>&1 | grep -E '"dmaz"' | cut -c1-260
done
