"""Summarise ncu evidence for profiles/:

  python scripts/ncu_summary.py --rep X.ncu-rep --launches launches.csv --out profiles/r01 [--traffic profiles/ncu_traffic.json]

* --rep: a `ncu --set full` capture; per kernel: duration, DRAM read/write
  bytes (-> per-launch traffic), DRAM/SM throughput, registers, smem, grid,
  occupancy and the top warp-stall reasons.  The per-stage traffic map used by
  bench.py's roofline.traffic is written to --traffic.
* --launches: the `--metrics gpu__time_duration.sum` launch list; per kernel
  family: launches and total / mean duration and its share of the summed time.

Kernel -> bench stage names follow the template arguments: pass_a_kernel<LZ,LT,MODE>
(MODE 0 = forward v, 1/2 = backward dz), pass_c_kernel<LZ,LT,EPI> (EPI 1 =
layer forward, 2 = layer backward)."""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import collections


def stage_of(name):
    m = re.match(r"(?:void )?(?:fno::)?(\w+?)(?:<(.*)>)?\(", name)
    base = m.group(1) if m else name.split("(")[0]
    targs = [re.sub(r"\(\w+\)", "", a).strip() for a in (m.group(2) or "").split(",")] if m else []
    if base in ("pass_a_kernel", "pass_a2_kernel") and len(targs) >= 3:       # <LZ, LT, MODE[, HALF]>
        return "fwd.pass_a" if targs[2] == "0" else "bwd.pass_a"
    if base == "pass_c_kernel" and len(targs) >= 3:                           # <LZ, LT, EPI>
        return {"0": "pass_c_u", "1": "fwd.pass_c", "2": "bwd.pass_c"}.get(targs[2], base)
    if base == "pass_c2_kernel" and len(targs) >= 4:                          # <LZ, LT, CP, EPI, HALF>
        return {"1": "fwd.pass_c", "2": "bwd.pass_c"}.get(targs[3], base)
    if base == "pass_c3_fwd_kernel":                                         # tcgen05 1x1 forward
        return "fwd.pass_c"
    if base == "pass_c4_kernel" and len(targs) >= 4:                          # <LZ, LT, CP, EPI, HALF, RAG>
        return {"0": "pass_c_u", "1": "fwd.pass_c", "2": "bwd.pass_c"}.get(targs[3], base)
    if base == "mix_fwd_kernel":
        return "fwd.mix"
    if base == "mix_bwd_kernel":
        return "bwd.mix"
    if base == "dw_partial_kernel":
        return "bwd.dw"
    return base


def stages_in_order(names):
    """stage_of over a launch sequence: a forward-mode pass C that follows a
    backward pass A is the split backward's dv leg (pass C family 5: the forward
    kernel run with W^T), i.e. bwd.pass_c"""
    out, in_bwd = [], False
    for n in names:
        st = stage_of(n)
        if st == "bwd.pass_a":
            in_bwd = True
        elif st == "fwd.pass_a":
            in_bwd = False
        if st == "fwd.pass_c" and in_bwd:
            st = "bwd.pass_c"
        out.append(st)
    return out


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def raw_rows(rep):
    """rep: an .ncu-rep, or the `--page raw --csv` export of one (optionally .gz)"""
    if rep.endswith(".csv") or rep.endswith(".csv.gz"):
        import gzip
        out = (gzip.open(rep, "rt") if rep.endswith(".gz") else open(rep)).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def to_bytes(v, unit):
    unit = unit.split("/")[0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return num(v) * scale


def to_us(v, unit):
    return num(v) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1e-3)


def summarise_rep(rep):
    rows, units = raw_rows(rep)
    stall_keys = [k for k in rows[0] if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")]
    res = []
    stages = stages_in_order([r.get("Kernel Name", "") for r in rows])
    for r, stage in zip(rows, stages):
        name = r.get("Kernel Name", "")
        rd = to_bytes(r["dram__bytes_read.sum"], units["dram__bytes_read.sum"])
        wr = to_bytes(r["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
        us = to_us(r["gpu__time_duration.sum"], units["gpu__time_duration.sum"])
        st = sorted(((num(r[k]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in stall_keys), reverse=True)
        tot = sum(v for v, _ in st if v == v) or 1.0
        res.append(dict(
            kernel=name[:160], stage=stage, duration_us=round(us, 2),
            dram_read_bytes=int(rd), dram_write_bytes=int(wr), dram_bytes=int(rd + wr),
            dram_gbs=round((rd + wr) / (us * 1e-6) / 1e9, 1) if us > 0 else None,
            dram_pct_peak=num(r.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "nan")),
            sm_pct_peak=num(r.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", "nan")),
            registers=int(num(r.get("launch__registers_per_thread", 0))),
            block=int(num(r.get("launch__block_size", 0))), grid=int(num(r.get("launch__grid_size", 0))),
            smem_per_block=int(to_bytes(r.get("launch__shared_mem_per_block", 0),
                                        units.get("launch__shared_mem_per_block", "byte"))),
            warps_active_pct=num(r.get("sm__warps_active.avg.pct_of_peak_sustained_active", "nan")),
            tensor_pipe_pct=num(r.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                                      r.get("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                                            "nan"))),
            issue_active_pct=num(r.get("smsp__issue_active.avg.pct_of_peak_sustained_active", "nan")),
            top_stalls=[(k, round(100 * v / tot, 1)) for v, k in st[:5]]))
    return res


def summarise_launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    fam = collections.OrderedDict()
    rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
    for r, st in zip(rows, stages_in_order([r["Kernel Name"] for r in rows])):
        us = to_us(r["Metric Value"], r["Metric Unit"])
        f = fam.setdefault(st, [0, 0.0])
        f[0] += 1
        f[1] += us
    tot = sum(v[1] for v in fam.values()) or 1.0
    return [dict(stage=k, launches=v[0], total_us=round(v[1], 1), mean_us=round(v[1] / v[0], 2),
                 share=round(v[1] / tot, 4)) for k, v in sorted(fam.items(), key=lambda kv: -kv[1][1])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    ap.add_argument("--config", default="c2", help="workload the capture ran (key of the traffic map)")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    md = []
    if a.rep:
        ks = summarise_rep(a.rep)
        json.dump(ks, open(os.path.join(a.out, "ncu_full_summary.json"), "w"), indent=1)
        md.append("## ncu --set full (one launch per kernel)\n")
        md.append("| stage | us | DRAM MB (r+w) | DRAM GB/s | DRAM % | SM % | issue % | tensor % | warps % | regs | "
                  "smem KB | grid x block | top stalls |")
        md.append("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
        for k in ks:
            stalls = ", ".join(f"{n} {p}%" for n, p in k["top_stalls"][:3])
            md.append(f"| {k['stage']} | {k['duration_us']} | {k['dram_bytes'] / 1e6:.1f} | {k['dram_gbs']} | "
                      f"{k['dram_pct_peak']:.1f} | {k['sm_pct_peak']:.1f} | {k['issue_active_pct']:.1f} | "
                      f"{k['tensor_pipe_pct']:.2f} | {k['warps_active_pct']:.1f} | {k['registers']} | "
                      f"{k['smem_per_block'] / 1024:.1f} | {k['grid']} x {k['block']} | {stalls} |")
        if a.traffic:
            allt = json.load(open(a.traffic)) if os.path.exists(a.traffic) else {}
            tr = {}
            for k in ks:   # last capture of a stage wins (all launches of a stage move the same bytes)
                tr[k["stage"]] = k["dram_bytes"]
            allt[a.config] = tr
            json.dump(allt, open(a.traffic, "w"), indent=1, sort_keys=True)
    if a.launches:
        fams = summarise_launches(a.launches)
        json.dump(fams, open(os.path.join(a.out, "ncu_launches_summary.json"), "w"), indent=1)
        md.append("\n## ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
        md.append("| stage | launches | total us | mean us | share |")
        md.append("|---|---|---|---|---|")
        for f in fams:
            md.append(f"| {f['stage']} | {f['launches']} | {f['total_us']} | {f['mean_us']} | {f['share']:.3f} |")
    open(os.path.join(a.out, "ncu_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
