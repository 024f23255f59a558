#!/bin/bash
# Pack iteration for the stream schedule: parity tests, sweep vs two-pass, optional ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { tail -30 gpurun_out/build.txt; exit 1; }
timeout 300 python tools/pack_sweep.py --schedules single_read --steps 20 ${SWEEP_ARGS} > gpurun_out/pack_sweep.txt 2>&1
echo "sweep rc=$?" >> gpurun_out/pack_sweep.txt
cat gpurun_out/pack_sweep.txt | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${PYTEST_K:-single_read}" > gpurun_out/pytest_pack.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_pack.txt
tail -15 gpurun_out/pytest_pack.txt
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_stream -s 0 -c 1 \
      -o gpurun_out/prof_pack_stream -f python tools/pack_sweep.py --schedules single_read --steps 2 > gpurun_out/ncu_stream.txt 2>&1
  tail -3 gpurun_out/ncu_stream.txt
fi
