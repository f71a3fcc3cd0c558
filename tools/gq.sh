#!/bin/bash
# quick GPU iteration: gpu tests (quiet) + bench headline + optional slow counts
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 100 --warmup 3 --no-sweep --no-cpu > gpurun_out/bq.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1]); print('value', round(d['value']), {k: round(v,4) for k,v in d['roofline']['launch_ms'].items()}, 'frac', round(d['roofline']['frac'],4))" || tail -5 gpurun_out/bq.log
