#!/bin/bash
# Pack iteration: pack parity tests (every schedule), schedule sweep, ncu of the cluster kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { tail -30 gpurun_out/build.txt; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pack" > gpurun_out/pytest_pack.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_pack.txt
tail -15 gpurun_out/pytest_pack.txt
timeout 300 python tools/pack_sweep.py --clusters ${CLUSTERS:-0,16,8,264,260} ${SWEEP_ARGS} > gpurun_out/pack_sweep.txt 2>&1
cat gpurun_out/pack_sweep.txt | tail -8
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_cluster -s 2 -c 1 \
      -o gpurun_out/prof_pack_cluster -f python tools/pack_sweep.py --clusters ${NCU_PARAM:-0} --steps 2 > gpurun_out/ncu_cluster.txt 2>&1
  tail -3 gpurun_out/ncu_cluster.txt
fi
