cd $GRAFT_REPO_ROOT
free -g | head -2
for lc in "" "--link-code"; do
  timeout 600 python tools/trace.py --functions 48 --mix 24,20,4 --duration-s 30 --pool-gb 6 --rate-lo 30 --rate-hi 150 $lc --out gpurun_out/trace_heavy${lc:+_coded}.json 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['link_code'], d['requests'], 'slo', d['slo_compliant_function_ratio'], 'met', d['request_deadline_ratio'], d['swap_kinds'], {k:(v['p50'],v['p98']) for k,v in d['latency_ms'].items()})"
done
