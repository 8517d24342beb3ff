import json, sys
d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/b_small.json').read().strip().split('\n')[-1])
print('%.3e' % d['value'], {k: round(v, 1) for k, v in d['stages_ms_per_step'].items()})
print({k: (round(v['ms_per_step'], 1), round(v['tflops'] or 0, 2)) for k, v in d['roofline']['per_kernel'].items()})
