#!/bin/bash
# A/B of environment settings in one box: bash profiles/ab_env.sh "VAR=a" "VAR=b" ...
mkdir -p gpurun_out
i=0
for e in "$@"; do
  i=$((i+1))
  env $e python bench.py $BENCH_ARGS --no-cpu-baseline --no-e2e --dropin-views 0 --steps 10 > gpurun_out/b_env$i.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/b_env$i.log') if l.startswith('{')][-1])
k=d['roofline']['kernel_ms_per_step']
print('$e', round(d['value'],1), k)" || tail -3 gpurun_out/b_env$i.log
done
