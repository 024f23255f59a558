#!/bin/bash
# Parity for every tiling + restore/pack timings on the narrow-tile-row layouts.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { tail -30 gpurun_out/build.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.txt
tail -15 gpurun_out/pytest_parity.txt
for lay in ${LAYS:-col1 a2b4 identity}; do
  for res in ${RESS:-R1080 R240}; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-fetch --layout $lay --res $res \
      > gpurun_out/bench_${lay}_${res}.json 2> gpurun_out/bench_${lay}_${res}.err
    python -c "import json; d=json.load(open('gpurun_out/bench_${lay}_${res}.json')); print('$lay $res restore', d['ms_per_step'], d['roofline']['frac'], 'pack', d.get('pack'))" || tail -5 gpurun_out/bench_${lay}_${res}.err
  done
done
