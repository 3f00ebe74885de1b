for c in C4 C3 C5 C2 C1; do python -c "
import json; d=json.loads(open('gpurun_out/all_$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$c', round(d['ms_per_step'],3), 'frac', round(r['frac'],4), 'k5', round(r['k5_ms_per_launch'],4), r.get('kernel'), 'e2e', (d.get('e2e') or {}).get('ms_per_step'))" 2>&1 | tail -1; done
