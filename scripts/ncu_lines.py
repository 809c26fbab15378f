"""Join an ncu sass-page CSV with nvdisasm line info: top source lines by
instructions executed and stall samples, per kernel.
usage: python scripts/ncu_lines.py <sass.csv> <cubin> <kernel-substring> [N]"""
import csv, re, subprocess, sys, collections

csvf, cubin, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# per function: list of (offset, file:line)
funcs = {}
cur = None; loc = None
for ln in dis.splitlines():
    m = re.match(r"^(\S+):$", ln.strip()) if ln and not ln.startswith(("\t", " ")) else None
    if ln.startswith(".text.") or (m and not ln.startswith(".")):
        name = ln.strip().rstrip(":").replace(".text.", "")
        cur = name; funcs.setdefault(cur, {}); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        loc = f"{m.group(1).split('/')[-1]}:{m.group(2)}"; continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(\S.*)", ln)
    if m and cur is not None:
        funcs[cur][int(m.group(1), 16)] = loc
rows = list(csv.reader(open(csvf)))
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name" and ksub in rows[i][1]:
        kname = rows[i][1]; hdr = rows[i + 1]; c = {h: k for k, h in enumerate(hdr)}
        body = []
        j = i + 2
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            body.append(rows[j]); j += 1
        # match function by instruction count
        base = int(body[0][0], 16)
        mm = re.search(r"(\w+)<([^>]*)>", kname)
        best = None
        if mm:
            targs = "".join(("Lb%sE" if "bool" in a else "Li%sE") % a.split(")")[-1].strip() for a in mm.group(2).split(","))
            key = mm.group(1) + "I" + targs
            cands = [kv for kv in funcs.items() if key in kv[0]]
            if cands: best = cands[0]
        if best is None:
            best = max(funcs.items(), key=lambda kv: (len(kv[1]) == len(body), -abs(len(kv[1]) - len(body))))
        lines = best[1]
        inst = collections.Counter(); samp = collections.Counter(); tot = 0; tots = 0
        for r in body:
            if len(r) < len(hdr): continue
            off = int(r[0], 16) - base
            L = lines.get(off, "?")
            n = float(r[c["Instructions Executed"]] or 0); s = float(r[c["Warp Stall Sampling (All Samples)"]] or 0)
            inst[L] += n; samp[L] += s; tot += n; tots += s
        print(f"== {kname[:80]}  ({best[0][:60]}, {len(body)} sass)  warp-inst {tot:.3g}")
        for L, n in sorted(inst.items(), key=lambda x: -samp[x[0]])[:N]:
            print(f"   {L:24s} inst {100*n/tot:5.1f}%   stall-samples {100*samp[L]/max(tots,1):5.1f}%")
        i = j
        break
    i += 1
