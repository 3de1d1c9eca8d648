for m in 127 0 126 125 123 119 111 95 63 1; do echo "mask $m"; FSW_PDL_MASK=$m timeout 120 python tools/full_gpu.py bert-base resnet50 2>&1 | grep warm; done
