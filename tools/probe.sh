set -x
nvidia-smi -q | grep -i -E "product name|decoder|encoder|clocks|max|sm " | head -40
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "Model name|Socket|Thread|Core"
ls /usr/lib/x86_64-linux-gnu | grep -E 'nvcuvid|nvidia-encode|libcuda'
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p, p.L2_cache_size if hasattr(p,'L2_cache_size') else '')"
python -c "import numba; print(numba.__version__)"
free -g
