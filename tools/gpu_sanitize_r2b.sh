# compute-sanitizer over the second-session kernels: v5 decode (SMZ / DMAZ), k_gemm_ws on every linear (push
# reduction over DSMEM), k_attention_tc.  No-overlap mode under the tool (libfsw detects it).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export FSW_GEMM_WS=2 FSW_ATTN_TC=1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_r2.py ws > gpurun_out/san_${t}_ws.log 2>&1; echo "$t rc=$?"
  tail -2 gpurun_out/san_${t}_ws.log
done
