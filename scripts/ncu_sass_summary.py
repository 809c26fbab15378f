"""Summarise an ncu --page source --print-source=sass csv: per kernel, opcode mix and stall reasons."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        kname = rows[i][1]
        hdr = rows[i + 1]
        j = i + 2
        body = []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            body.append(rows[j]); j += 1
        c = {h: k for k, h in enumerate(hdr)}
        ops = collections.Counter(); stalls = collections.Counter(); samp = collections.Counter()
        tot_inst = 0
        for r in body:
            if len(r) < len(hdr): continue
            src = r[c["Source"]].strip()
            op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
            op = op.split(".")[0]
            n = float(r[c["Instructions Executed"]] or 0)
            ops[op] += n; tot_inst += n
            samp[op] += float(r[c["Warp Stall Sampling (All Samples)"]] or 0)
            for h, k in c.items():
                if h.startswith("stall_"):
                    try: stalls[h] += float(r[k] or 0)
                    except ValueError: pass
        print(f"== {kname[:90]}  warp-instructions={tot_inst:.3g}")
        for op, n in ops.most_common(22):
            print(f"   {op:10s} {n:12.4g} {100*n/tot_inst:5.1f}%   stall-samples {samp[op]:.0f}")
        ts = sum(stalls.values())
        print("   stalls:", ", ".join(f"{k[6:]}={100*v/ts:.1f}%" for k, v in stalls.most_common(8)))
        i = j
    else:
        i += 1
