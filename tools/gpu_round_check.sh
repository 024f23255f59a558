#!/bin/bash
# Round-end style check on one B200: pytest -m gpu, smoke, default bench, reference arm.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/rc; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1 || { tail -30 $O/build.txt; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
tail -c 600 $O/bench_default.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
tail -c 300 $O/bench_reference.json
