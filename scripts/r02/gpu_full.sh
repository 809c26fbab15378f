#!/bin/bash
# full GPU suite, smoke, and the default bench line (c3) + c2
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-full}
timeout 1800 python -m pytest tests -q -m gpu -x > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_$TAG.log
timeout 900 python bench.py > $O/bench_default_$TAG.json 2> $O/bench_default_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2_$TAG.json 2> $O/bench_c2_$TAG.err; echo "bench c2 rc=$?"
python scripts/show_bench.py $O/bench_default_$TAG.json $O/bench_c2_$TAG.json
