#!/bin/bash
# Box probe for SURVEY §7 step 0 / VERDICT f4: NVDEC engines and cuvid availability.
mkdir -p gpurun_out
{
echo "== nvidia-smi -q (decoder/encoder/clocks)"
nvidia-smi -q | grep -iE -A3 "Product Name|Decoder|Encoder|JPEG|OFA|Max Clocks|Utilization" | head -80
echo "== nvidia-smi --query"
nvidia-smi --query-gpu=name,driver_version,utilization.decoder,utilization.encoder,clocks.max.sm --format=csv
echo "== ldconfig -p | grep nvcuvid/nvidia-encode"
ldconfig -p | grep -E "nvcuvid|nvidia-encode|libnvidia-opticalflow" || echo "(none in ldconfig)"
echo "== find libnvcuvid"
find / -xdev \( -name 'libnvcuvid*' -o -name 'libnvidia-encode*' -o -name 'nvcuvid.h' -o -name 'cuviddec.h' \) 2>/dev/null | head
echo "== nproc / cpu"
nproc; lscpu | grep -E "Model name|Socket|Thread|Core"
echo "== torch props"
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.L2_cache_size if hasattr(p,'L2_cache_size') else '')"
} > gpurun_out/probe_box.txt 2>&1
cat gpurun_out/probe_box.txt
