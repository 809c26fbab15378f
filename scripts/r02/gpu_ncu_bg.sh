#!/bin/bash
O=gpurun_out/r02bg; mkdir -p $O
CMD="python bench.py --config c3 --steps 2 --warmup 1 --layers 1 --no-cpu-baseline --no-phases --no-graph"
$CMD > $O/plain.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k 'regex:pass_c4' -s 6 -c 6 --csv --log-file $O/bg.csv $CMD > $O/ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.DictReader([l for l in open('gpurun_out/r02bg/bg.csv') if l.startswith('"')]))
for r in rows:
    print(r['Kernel Name'][:60], r['Metric Name'], r['Metric Value'], r['Metric Unit'])
PY
