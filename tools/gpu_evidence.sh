#!/bin/bash
# Round evidence on one B200: default bench line, other configs / layouts, pack
# schedule sweep, ncu launch list and --set full captures of the hot kernels.
# Outputs under gpurun_out/ev/ (copied into profiles/<round>/ by hand).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/ev; mkdir -p $O
python -m paper_2602_09725_b200.build > $O/build.txt 2>&1 || { tail -30 $O/build.txt; exit 1; }
nvidia-smi -q > $O/nvidia_smi_q.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
if [ -z "$SKIP_BENCH" ]; then
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
for cfg in "--layout paper" "--layout col1" "--layout a2b4" "--res R240" \
           "--model qwen2.5-7b --tokens 131072" "--model llama3-70b --tokens 81920"; do
  tag=$(echo "$cfg" | tr -d '-' | tr ' ' '_')
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-fetch $cfg \
     > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "$tag rc=$?"
done
timeout 300 python tools/pack_sweep.py --schedules single_read,single_read:16 --steps 20 > $O/pack_sweep.jsonl 2>&1
timeout 300 python tools/pack_sweep.py --schedules single_read --steps 20 --layout col1 > $O/pack_sweep_col1.jsonl 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu && timeout 120 /tmp/tma_probe > $O/tma_probe.txt 2>&1
timeout 300 python tools/head_probe.py > $O/head_probe.jsonl 2>&1
timeout 600 python tools/fed_probe.py > $O/fed_probe.txt 2>&1
fi
if [ -z "$SKIP_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu > $O/ncu_launch_stdout.txt 2>&1
echo "launch list rc=$?"
FULL="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-fetch"
for k in restore_fast absmax_fast pack_fast; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o $O/prof_$k -f $FULL > $O/ncu_${k}.txt 2>&1; echo "$k rc=$?"
done
# the band kernels run 2 launches per step: capture both launches of one step
for k in restore_band pack_band; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 2 \
      -o $O/prof_${k}_col1 -f $FULL --layout col1 > $O/ncu_${k}.txt 2>&1; echo "$k rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pack_stream -s 0 -c 1 \
    -o $O/prof_pack_stream -f python tools/pack_sweep.py --schedules single_read --steps 2 > $O/ncu_pack_stream.txt 2>&1; echo "pack_stream rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rc_decode_kernel -s 0 -c 1 \
    -o $O/prof_rc_decode_fed -f python tools/fed_probe.py --quick > $O/ncu_fed.txt 2>&1; echo "fed rc=$?"
# the plain range decoder over all of C2's planes in one launch (device-resident bytes)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rc_decode -s 0 -c 1 \
    -o $O/prof_rc_decode -f python tools/rc_probe.py > $O/ncu_rc_decode.txt 2>&1; echo "rc_decode rc=$?"
timeout 600 python tools/rc_probe.py > $O/rc_probe.txt 2>&1
timeout 600 python tools/rc_probe.py --pinned > $O/rc_probe_fed.txt 2>&1
fi

# summaries on the box (the reports themselves stay there: gpurun brings back <= 64 MiB)
if [ -z "$SKIP_NCU" ]; then
K="llama3-8b/32768/identity/R1080/page16/req1/balanced/n1"
KC="llama3-8b/32768/col1/R1080/page16/req1/balanced/n1"
rm -rf profiles/evx
python tools/ncu_summary.py evx --config $K $O/launches.csv $O/prof_restore_fast.ncu-rep \
    $O/prof_absmax_fast.ncu-rep $O/prof_pack_fast.ncu-rep $O/prof_pack_stream.ncu-rep \
    $O/prof_rc_decode.ncu-rep $O/prof_rc_decode_fed.ncu-rep > $O/summ.txt 2>&1
python tools/ncu_summary.py evx --config $KC $O/prof_restore_band_col1.ncu-rep \
    $O/prof_pack_band_col1.ncu-rep >> $O/summ.txt 2>&1
mkdir -p $O/summ && cp profiles/evx/* $O/summ/ && cp $O/launches.csv $O/summ/launches_raw.csv
rm -f $O/*.ncu-rep
fi
ls -la $O
