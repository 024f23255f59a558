cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/probe_box.sh > /dev/null 2>&1
bash tools/gpu_check.sh
timeout 300 python tools/pack_sweep.py --slabs 8,16,32,64 > gpurun_out/pack_sweep.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/smoke.txt; tail -2 gpurun_out/bench.txt | cut -c1-600; cat gpurun_out/pack_sweep.txt | tail -6
