# Heavy/light policy on the heavy Poisson trace (48 functions, link-coded): SLO-slack classes
# (theta 0.05) vs every model heavy (the paper's execution-relative rule at batch 1).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for mode in "slo" "allheavy"; do
  extra=""; [ "$mode" = "allheavy" ] && extra="--all-heavy"
  timeout 600 python tools/trace.py --functions 48 --mix 24,20,4 --duration-s 30 --pool-gb 6 --rate-lo 30 --rate-hi 150 --link-code $extra --out gpurun_out/trace_classes_${mode}.json 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$mode', d['requests'], 'slo', d['slo_compliant_function_ratio'], 'met', d['request_deadline_ratio'], d['swap_kinds'], 'heavy', d['heavy_models_after'], 'evict', d['eviction_mix'], {k:(v['p50'],v['p98']) for k,v in d['latency_ms'].items()})"
done
