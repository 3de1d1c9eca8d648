# Round-2 final evidence (second session): the default bench line and the reference arm, the ncu launch list of
# the bench command, --set full of the resident BERT-base GEMMs (k_gemm_ws) and of the v5 DMAZ decode.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_r2c_reference.json 2> gpurun_out/bench_r2c_reference.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_default_r2c.csv \
  python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline --no-extras > gpurun_out/ncu_bench_r2c.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py gpurun_out/launches_bench_default_r2c.csv > gpurun_out/launches_bench_default_r2c_summary.txt; head -12 gpurun_out/launches_bench_default_r2c_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 49 -c 4 -o gpurun_out/prof_gemm_bert_resident_r2c \
  python tools/profile_target.py bert-base 1 sm > gpurun_out/ncu_gemm_r2c.log 2>&1; echo "ncu gemm rc=$?"
ncu -i gpurun_out/prof_gemm_bert_resident_r2c.ncu-rep --page raw --csv > gpurun_out/prof_gemm_bert_resident_r2c.raw.csv 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/bench_r2c.json')); print({k:d[k] for k in ['value','p99_ms','resident_p50_ms','link_wire_gbs','gpu_launches','clocks']}, d['e2e']['value'], d['roofline']['frac'], d['native_torch_resident_ms'])
print({k:(v.get('p50_ms'),v.get('resident_p50_ms')) for k,v in d['configs_1gpu'].items()})
r=json.load(open('gpurun_out/bench_r2c_reference.json')); print(r['impl'], r['value'], r['unit'])"
