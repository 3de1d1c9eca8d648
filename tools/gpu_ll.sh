cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bert_warm.csv python tools/profile_target.py bert-base 2 dmaz > /dev/null 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gpt2l_warm.csv python tools/profile_target.py gpt2-2L 2 > /dev/null 2>&1; echo rc=$?
