#!/bin/bash
# One line per workload: windows/s, ms/step and the dominant launch's HBM fraction.
for w in ${@:-swin_t_fwd swin_t_fwdbwd swin_b_fwdbwd large_sweep}; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu --no-e2e --no-extra 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']
        print('$w', f\"{d['value']:.4g} {d['unit']} ms={d['ms_per_step']:.4f} step_frac={r.get('step_frac',0):.3f} dom_frac={r['frac']:.3f}\", {k:(round(v['ms'],4),round(v['GB/s'])) for k,v in r.get('launches',{}).items()})
"
done
