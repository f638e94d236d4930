import json,sys
for l in sys.stdin:
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); st=d['steps']
    print(d['config']['workload'], round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), {k:round(v['ms']/st,3) for k,v in d.get('kernels',{}).items()}, 'e2e', (d.get('e2e') or {}).get('value'))
