#!/bin/bash
# Standard measurement batch on the GPU box: quick parity, bench, per-model timings, launch lists.
set -x
timeout 300 python tools/debug_ops.py 2>&1 | grep -v "row" | tail -12
timeout 300 python tools/quick_gpu.py 2>&1 | tail -6
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_quick.json
cat gpurun_out/bench_quick.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','p99_ms','resident_p50_ms','swap_p50_ms','compute_tail_p50_ms','host_to_hbm_gbs','frac_of_pipelined_roofline']})"
timeout 300 python tools/full_gpu.py resnet50 mlp gpt2-2L 2>&1 | tail -20
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bert4.csv python tools/profile_target.py bert-base 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_resnet4.csv python tools/profile_target.py resnet50 1 > /dev/null 2>&1
