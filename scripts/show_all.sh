for c in C4 C3 C5 C2 C1; do python -c "
import json; d=json.loads(open('gpurun_out/all_$c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$c', round(d['ms_per_step'],3), 'frac', round(r['frac'],4), 'k5', r.get('isolated',{}).get('k5_ms_per_launch', r.get('k5_ms_per_launch')), r.get('kernel'))" 2>&1 | tail -1; done
