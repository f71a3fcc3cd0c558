#!/bin/bash
# quick GPU check: parity report + bench summary line
python tests/diagnostics/parity_report.py C4 C5 C2 C1 2>&1 | grep case | python -c "
import json,sys
bad=0; n=0
for l in sys.stdin:
    d=json.loads(l); n+=1; bad+=not d['ok']; print(d['case'], d['form'][:12], 'ok' if d['ok'] else 'FAIL', 'ang %.1e res %.1e curv %.1e st %d' % (d['max_normal_rad'], d['max_residual_rel'], d['max_curvature_rel'], d['status_mismatch']))
print('PARITY', n - bad, 'of', n, 'ok')"
python bench.py --steps 50 --warmup 3 --no-cpu > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('value', round(d['value']), 'launch_ms', {k: round(v,4) for k,v in d['roofline']['launch_ms'].items()}, 'frac', round(d['roofline']['frac'],4))"
