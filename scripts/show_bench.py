import json, sys
d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench.json').read().strip().splitlines()[-1])
print(f"value={d['value']:.4g} ms/step={d['ms_per_step']} e2e={d['e2e']['value']:.4g} launches={d.get('gpu_launches')} clocks={d.get('clocks')}")
print("roofline:", d.get('roofline'))
for k, v in sorted(d.get('stages', {}).items(), key=lambda x: -x[1]['ms_per_step']):
    print(f"  {k:18s} {v['ms_per_step']:8.3f} ms/step  {v['GBps']} GB/s")
if d.get('cpu_baseline'): print("cpu:", d['cpu_baseline']['value'], d['cpu_baseline']['cores'])
