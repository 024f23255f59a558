#!/bin/bash
# Fetch-to-ready leg at two resolution classes + ncu of the KVFC decode kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
for res in ${RESES:-R1080 R240}; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --res $res > gpurun_out/fetch_$res.json 2> gpurun_out/fetch_$res.err
  python -c "import json; d=json.load(open('gpurun_out/fetch_$res.json')); print('$res', d['fetch_to_ready'], d['ms_per_step'])" || tail -3 gpurun_out/fetch_$res.err
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rc_decode|recon_kernel" -c 2 \
     -o gpurun_out/prof_decode -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --res ${NCU_RES:-R1080} > gpurun_out/ncu_decode.txt 2>&1
  tail -2 gpurun_out/ncu_decode.txt
fi
