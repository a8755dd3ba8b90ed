#!/bin/bash
# A/B of library variants on the drop-in call: bash profiles/ab_dropin.sh WORKLOAD lib1.so lib2.so ...
w=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  SDGR_LIB=$lib python bench.py --workload $w --no-cpu-baseline --no-e2e --dropin-views 30 --steps 5 > gpurun_out/bd_$lib.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bd_$lib.log') if l.startswith('{')][-1]); e=d['e2e_dropin']
print('$w $lib', round(d['value'],1), 'dropin', round(e['value'],1), 'median_ms', round(e['median_call_ms'],3))"
done
