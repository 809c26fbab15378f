#!/bin/bash
# One GPU call that produces the round's evidence (run via gpurun from the repo root):
#   gpu tests (incl. slow full-size), smoke(), bench (default command), the ncu
#   launch list of the bench command and one `ncu --set full` capture of every
#   kernel of one layer step.  Summarise afterwards, here:
#   python scripts/ncu_summary.py --rep gpurun_out/prof_$TAG.ncu-rep \
#       --launches gpurun_out/launches_$TAG.csv --out profiles/$TAG --traffic profiles/ncu_traffic.json
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1
rc=$?; echo "plain rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pass_|b_|mix_|rowsum" -c 1000 --csv \
      --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?"
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"pass_|b_|mix_|rowsum" -s 15 -c 15 \
      -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --layers 1 --no-cpu-baseline \
      > gpurun_out/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?"
fi
