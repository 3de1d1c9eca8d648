# Link format v4 final check: full GPU suite, smoke, bench lines, engine table, paper table.
bash tools/gpu_verify.sh
cd $GRAFT_REPO_ROOT
timeout 900 python tools/linkcode_bench.py mlp resnet50 bert-base gpt2-xl --reps 20 > gpurun_out/linkcode_v4.jsonl 2>&1
timeout 600 python tools/paper_table.py resnet50 resnet101 resnet152 bert-base bert-large > gpurun_out/paper_table_v4.txt 2>&1
tail -5 gpurun_out/paper_table_v4.txt | cut -c1-250
