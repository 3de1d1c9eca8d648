# In-graph tiling sweep of the per-op k_gemm on resident BERT-base (FSW_GEMM_FORCE applies to the linears
# whose modelled tiling is not split-K: QKV, O-proj, FFN1): resident p50 and the per-op critical path.
cd ${GRAFT_REPO_ROOT:-.}
for f in "" "16:2:1" "32:2:1" "16:3:1" "32:3:1" "64:2:1" "16:4:1" "32:4:1" "16:2:0" "32:2:0"; do
  echo "FSW_GEMM_FORCE=$f"
  FSW_GEMM_FORCE=$f timeout 120 python tools/timeline.py --model bert-base --reps 10 2>&1 | grep -E "resident invoke device|critical-path"
done
