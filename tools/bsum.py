import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(d['config'].get('workload'), round(d['ms_per_step'],3), round(d['value'],1), d['unit'], 'frac', (d.get('roofline') or {}).get('frac'))
