#!/bin/bash
# Pack iteration: parity tests for pack, then bench timings per pack mode.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pack" > gpurun_out/pytest_pack.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_pack.txt
tail -5 gpurun_out/pytest_pack.txt
for mode in ${MODES:-team twopass}; do
  KVF_PACK_MODE=${mode%%:*} KVF_TEAM_LAG=${mode#*:} timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu ${BENCH_ARGS} \
    > gpurun_out/pack_${mode}.json 2> gpurun_out/pack_${mode}.err
  python -c "import json; d=json.load(open('gpurun_out/pack_${mode}.json')); print('$mode', d['pack'])" || tail -5 gpurun_out/pack_${mode}.err
done
if [ -n "$NCU" ]; then
  KVF_PACK_MODE=team timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_team -s 1 -c 1 \
      -o gpurun_out/prof_pack_team -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_team.txt 2>&1
  tail -3 gpurun_out/ncu_team.txt
fi
