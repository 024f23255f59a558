#!/bin/bash
# ncu evidence for profiles/<round>/: the launch list of the bench command
# (serialised, cold-cache: compare shares, not absolutes) and one --set full
# capture per hot kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { echo BUILD FAILED; cat gpurun_out/build.txt; exit 1; }
CMD="python bench.py --steps 10 --warmup 3 --no-cpu ${BENCH_ARGS}"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch_stdout.txt 2>&1
echo "launch list rc=$?"
FULL="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS}"
for k in ${KERNELS:-restore_fast absmax_fast pack_fast rc_decode recon_kernel rc_encode}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_$k -f $FULL > gpurun_out/ncu_${k}_stdout.txt 2>&1
  echo "$k rc=$?"
done
ls gpurun_out/*.ncu-rep
