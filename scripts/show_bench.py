"""Print the headline, roofline and per-stage table of bench.py JSON lines."""
import json
import sys

for path in sys.argv[1:] or ["gpurun_out/bench.json"]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    print(f"== {path}: value={d['value']:.4g} ms/step={d['ms_per_step']} e2e={d['e2e']['value']:.4g} "
          f"launches={d.get('gpu_launches')} clocks={d.get('clocks')}")
    r = d.get("roofline") or {}
    print(f"   dominant {r.get('kernel')} frac={r.get('frac')} avg_us={r.get('avg_launch_us')}")
    sr = d.get("step_roofline") or {}
    print(f"   step roofline t_roof={sr.get('t_roof_sum_ms')} ms frac_sum={sr.get('frac_sum')}")
    for k, v in sorted(d.get("stages", {}).items(), key=lambda x: -x[1]["ms_per_step"]):
        print(f"     {k:18s} {v['ms_per_step']:8.3f} ms/step  {v['GBps']} GB/s")
