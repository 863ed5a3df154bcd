import json, sys
p = sys.argv[1] if len(sys.argv) > 1 else '/root/repo/gpurun_out/bench.log'
l = [x for x in open(p) if x.startswith('{')]
if not l:
    print(open(p).read()[-3000:]); sys.exit()
d = json.loads(l[-1])
print("value", round(d['value'], 1), "upd_ms", round(d['update_ms_per_step'], 3), "ms/step", round(d['ms_per_step'], 2))
print({k: round(v, 3) for k, v in d['phase_ms'].items()})
for k, v in d['kernels'].items():
    print(f"  {k:10s} ms/step {v['ms_per_step']:8.3f} launches {v['launches_per_step']:6.0f} GB/s {v['alg_GBps'] or 0:8.1f} frac {v['frac_of_peak'] or 0:.3f}")
print(d['roofline'])
print({k: (round(v, 1) if isinstance(v, float) else v) for k, v in d['queries'].items()})
print(d['clocks'], d.get('gpu_launches'))
