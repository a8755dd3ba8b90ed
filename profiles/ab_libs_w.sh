#!/bin/bash
# A/B of library variants over workloads: bash profiles/ab_libs_w.sh "c4 c2 c3" lib1.so lib2.so ...
ws=$1; shift
mkdir -p gpurun_out
for w in $ws; do for lib in "$@"; do
  SDGR_LIB=$lib python bench.py --workload $w --no-cpu-baseline --no-e2e --dropin-views 0 --steps 10 > gpurun_out/bw_$lib.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bw_$lib.log') if l.startswith('{')][-1])
print('$w $lib', round(d['value'],1), round(d['preprocess_sort_roofline']['frac_comp_plane_only'],4))"
done; done
