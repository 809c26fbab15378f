"""Attribute ncu SASS-level stall samples / instruction counts to the
enclosing source line of a chosen file (so inlined helpers such as mbarrier
waits are charged to their call sites), optionally bucketed by line ranges.
usage: python scripts/ncu_callsites.py <sass.csv> <cubin> <mangled-substring> <file> [a-b:name ...]"""
import collections, csv, re, subprocess, sys

csvf, cubin, fsub, fname = sys.argv[1:5]
ranges = []
for a in sys.argv[5:]:
    lohi, name = a.split(":")
    lo, hi = map(int, lohi.split("-"))
    ranges.append((lo, hi, name))
rows = list(csv.reader(open(csvf)))
hdr = rows[1]; c = {h: i for i, h in enumerate(hdr)}
body = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name": break
    body.append(r)
base = int(body[0][0], 16)
lines = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith(".text.") and fsub in l][0]
locs = {}; loc = None; last = None
for l in lines[start + 1:]:
    if l.startswith(".text."): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        f = m.group(1).split("/")[-1]; loc = f"{f}:{m.group(2)}"
        if f == fname: last = int(m.group(2))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m: locs[int(m.group(1), 16)] = (loc, last)
st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
site = collections.Counter(); inst = collections.Counter(); grp = collections.defaultdict(collections.Counter)
ginst = collections.Counter(); tot = 0
for r in body:
    off = int(r[0], 16) - base
    L, ln = locs.get(off, (None, None))
    s = float(r[c["Warp Stall Sampling (All Samples)"]] or 0); n = float(r[c["Instructions Executed"]] or 0)
    tot += s
    site[(ln, L)] += s; inst[(ln, L)] += n
    g = next((nm for lo, hi, nm in ranges if ln is not None and lo <= ln <= hi), "other")
    ginst[g] += n
    for h in st: grp[g][h] += float(r[c[h]] or 0)
print("top call sites by stall samples (enclosing line, innermost line):")
for k, v in site.most_common(15):
    print(f"  {str(k[0]):>5} {str(k[1]):28s} stall {100*v/tot:5.1f}%  warp-inst {inst[k]:.3g}")
if ranges:
    gt = sum(sum(v.values()) for v in grp.values())
    for g, v in grp.items():
        s = sum(v.values())
        print(f"{g:12s} warp-inst {ginst[g]:.3g} stall-share {100*s/gt:5.1f}%  " +
              ", ".join(f"{k[6:]} {100*x/max(s,1):.0f}%" for k, x in v.most_common(5)))
