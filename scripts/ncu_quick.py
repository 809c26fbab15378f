"""Quick ncu report digest: key SOL / issue / occupancy metrics, stall totals
and per-source-region instruction shares.
usage: python scripts/ncu_quick.py <rep.ncu-rep> [kernel-id]"""
import csv, collections, io, subprocess, sys

rep = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else None
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(det)))
h = r[0]; c = {x: i for i, x in enumerate(h)}
want = {"Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "L1/TEX Cache Throughput", "Eligible Warps Per Scheduler", "Grid Size"}
for row in r[1:]:
    if kid is not None and row[c["ID"]] != kid: continue
    if row[c["Metric Name"]] in want:
        print(row[c["ID"]], row[c["Kernel Name"]][:40], row[c["Metric Name"]], row[c["Metric Value"]], row[c["Metric Unit"]])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; cc = {x: i for i, x in enumerate(hdr)}
st = [x for x in hdr if x.startswith("stall_") and "Not Issued" not in x]
tot = collections.Counter(); inst = 0
for rr in rows[2:]:
    if rr and rr[0] == "Kernel Name": break
    if len(rr) < len(hdr): continue
    inst += float(rr[cc["Instructions Executed"]] or 0)
    for x in st: tot[x] += float(rr[cc[x]] or 0)
s = sum(tot.values())
print("warp-instructions executed (first kernel):", f"{inst:.4g}")
print("stalls:", ", ".join(f"{k[6:]} {100*v/s:.1f}%" for k, v in tot.most_common(9)))
