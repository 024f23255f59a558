#!/bin/bash
# Sharded product test, bench (ours + reference arm), and a 2-rank run on one GPU.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m paper_2602_09725_b200.build > gpurun_out/build.txt 2>&1 || { tail -30 gpurun_out/build.txt; exit 1; }
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/pytest_shard.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_shard.txt; tail -4 gpurun_out/pytest_shard.txt
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$?"; tail -3 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
   bench.py --gpus 2 --steps 20 --warmup 5 --dist-backend gloo --no-e2e --no-fetch --no-cpu > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "n2 rc=$?"; tail -3 gpurun_out/bench_n2.err
