#!/bin/bash
# quick GPU iteration: gpu tests (quiet) + bench headline
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 100 --warmup 3 --no-sweep --no-cpu > gpurun_out/bq.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1]); print('value', round(d['value']), 'ms_step', round(d['ms_per_step'],4), 'launches', d['roofline']['launches_per_step'], 'frac', round(d['roofline']['frac'],4))" || tail -5 gpurun_out/bq.log
