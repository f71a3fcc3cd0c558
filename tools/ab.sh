#!/bin/bash
# A/B timing of library variants: ab.sh name[:ENV=VAL] ... (name main = in-tree library)
for spec in "$@"; do
  name=${spec%%:*}; envs=""; [ "$spec" != "$name" ] && envs=${spec#*:}
  lib=$PWD/paper_2103_06644_b200/librangefit_b200.so; [ "$name" != main ] && lib=$PWD/paper_2103_06644_b200/librangefit_b200_$name.so
  env RF_LIB_PATH=$lib $envs python bench.py --steps 200 --warmup 5 --no-sweep --no-cpu > gpurun_out/ab_$name.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$name.log').read().strip().splitlines()[-1]); print('$spec', 'value', round(d['value']), 'ms_step', round(d['ms_per_step'],4), 'launches', d['roofline']['launches_per_step'])" || tail -3 gpurun_out/ab_$name.log
done
