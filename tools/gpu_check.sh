#!/bin/bash
# One GPU round: parity tests, smoke, a short bench.  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { echo BUILD FAILED; cat gpurun_out/build.txt; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.txt 2>&1
echo "bench rc=$?" >> gpurun_out/bench.txt
