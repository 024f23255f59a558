#!/bin/bash
# ncu evidence: launch list (serialised, cold) + one --set full capture per hot kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { echo BUILD FAILED; cat gpurun_out/build.txt; exit 1; }
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu ${BENCH_ARGS}"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch_stdout.txt 2>&1
for k in ${KERNELS:-restore_fast pack_fast absmax_fast}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$k -f $CMD > gpurun_out/ncu_${k}_stdout.txt 2>&1
done
ls -la gpurun_out
