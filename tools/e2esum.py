import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); e=d.get('e2e') or {}
        print(d['config'].get('workload'), 'ms', round(d['ms_per_step'],3), 'value', round(d['value'],1), 'e2e_ms', round(e.get('ms_per_step',0),2), 'e2e', round(e.get('value',0),1))
