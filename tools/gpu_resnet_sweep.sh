# ResNet-50 cold-invoke engine sweep and device timelines (SMZ vs DMAZ) on one B200.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 900 python tools/resnet_sweep.py resnet50 > gpurun_out/resnet_sweep.txt 2>&1; echo "sweep rc=$?"
timeout 300 python tools/timeline.py --model resnet50 --engine 3 --out gpurun_out/timeline_resnet50_smz_r2e.txt > /dev/null 2>&1; echo "tl smz rc=$?"
timeout 300 python tools/timeline.py --model resnet50 --engine 4 --out gpurun_out/timeline_resnet50_dmaz_r2e.txt > /dev/null 2>&1; echo "tl dmaz rc=$?"
cat gpurun_out/resnet_sweep.txt | tail -80
