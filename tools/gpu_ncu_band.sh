#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { tail -30 gpurun_out/build.txt; exit 1; }
for k in restore_band pack_band; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/prof_$k -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-fetch --layout ${LAY:-col1} > gpurun_out/ncu_$k.txt 2>&1
tail -2 gpurun_out/ncu_$k.txt
done
