cd $GRAFT_REPO_ROOT
for lc in "" "--link-code"; do
  timeout 900 python tools/trace.py --functions 200 --mix 100,80,20 --duration-s 120 --pool-gb 8 --rate-lo 5 --rate-hi 30 $lc --out gpurun_out/trace200${lc:+_coded}.json 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['link_code'], d['requests'], 'slo', d['slo_compliant_function_ratio'], 'met', d['request_deadline_ratio'], d['swap_kinds'], {k:(v['p50'],v['p98']) for k,v in d['latency_ms'].items()})"
done
