"""Top CUDA source lines by warp-stall samples from an ncu report
(`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`).

    python scripts/ncu_cuda_lines.py X.ncu-rep [kernel-substring] [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
if rep.endswith(".csv") or rep.endswith(".csv.gz"):   # the source page exported on the GPU box
    import gzip
    out = (gzip.open(rep, "rt") if rep.endswith(".gz") else open(rep)).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per = {}
fpath = func = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or func is None or ksub not in func or len(r) < 5 or r[2] != "-":
        continue
    try:
        samp = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        inst = int(r[hdr["Instructions Executed"]] or 0)
    except (ValueError, KeyError):
        continue
    d = per.setdefault(func, {})
    d[(fpath, int(r[0]))] = (samp, inst, r[1].strip()[:90])
for func, d in per.items():
    tot = sum(v[0] for v in d.values()) or 1
    toti = sum(v[1] for v in d.values()) or 1
    print(f"== {func[:110]}  samples {tot}")
    for (f, ln), (s, i, src) in sorted(d.items(), key=lambda kv: -kv[1][0])[:N]:
        print(f"  {s / tot * 100:5.1f}%  inst {i / toti * 100:5.1f}%  {f}:{ln:<5d} {src}")
