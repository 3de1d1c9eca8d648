# DMA group taper fraction sweep (FSW_DMA_TAPER): cold p50 of ResNet-50 / BERT-base / MLP
for f in 0.5 0.67 0.75 0.85 0.95; do
  echo "taper $f"; FSW_DMA_TAPER=$f timeout 200 python tools/full_gpu.py resnet50 bert-base 2>&1 | grep -E "cold\[default\]|^[a-z]"
done
