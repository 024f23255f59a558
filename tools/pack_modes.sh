#!/bin/bash
# Compare pack schedules (two-pass default vs KVF_PACK_MODE=fused) on the bench workload.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
for mode in ${MODES:-twopass fused l2}; do
  for lay in ${LAYS:-identity paper}; do
    KVF_PACK_MODE=$mode timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --layout $lay \
      > gpurun_out/pack_${mode}_${lay}.json 2> gpurun_out/pack_${mode}_${lay}.err
  done
done
KVF_PACK_MODE=${NCU_MODE:-l2} timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv \
    --log-file gpurun_out/launches_${NCU_MODE:-l2}.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
