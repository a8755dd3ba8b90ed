#!/bin/bash
# A/B of bench.py arguments: bash profiles/ab_args.sh "--lanes 8" "--lanes 12" ...
mkdir -p gpurun_out
for a in "$@"; do
  python bench.py $a --no-cpu-baseline --no-e2e --dropin-views 0 --steps 10 > gpurun_out/ba.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/ba.log') if l.startswith('{')][-1])
print('$a', round(d['value'],1))" || tail -2 gpurun_out/ba.log
done
