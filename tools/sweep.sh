#!/bin/bash
# config sweep summary (bench.py's informational sweep)
python bench.py --steps 30 --warmup 3 --no-cpu --no-parity > gpurun_out/bsw.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bsw.log').read().strip().splitlines()[-1])
print('value', round(d['value']))
print(' '.join(f\"{k}:{round(v['Mpixel_fits_per_s']/1e3,1)}k\" for k,v in d['sweep'].items()))"
