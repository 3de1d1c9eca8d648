#!/bin/bash
# Round-1 measurement batch on the GPU box: discovery, GPU tests, bench, launch lists, ncu captures.
mkdir -p gpurun_out
bash tools/box_discovery.sh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
timeout 600 python tools/full_gpu.py resnet50 mlp --sweep > gpurun_out/full_gpu.log 2>&1
# launch list of one no-overlap cold invoke + 2 warm invokes (bert-base)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bert.csv python tools/profile_target.py bert-base 2 > /dev/null 2>&1
# swap kernel: full set + PCIe/sysmem counters (swap-only: no-overlap cold invoke)
timeout 900 ncu --set full --clock-control none --import-source on --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,syslts__t_sectors_aperture_sysmem_op_read.sum \
  -k regex:k_swap -c 1 -o gpurun_out/prof_swap python tools/profile_target.py bert-base 0 > gpurun_out/ncu_swap.log 2>&1
# top GEMM (resident)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 20 -c 2 -o gpurun_out/prof_gemm python tools/profile_target.py bert-base 1 > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
