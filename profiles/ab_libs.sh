#!/bin/bash
# A/B of library variants in one box: bash profiles/ab_libs.sh KERNEL lib1.so lib2.so ...
# (variants built with SDGR_EXTRA_FLAGS / SDGR_BUILD_SUFFIX / SDGR_LIB_NAME, see csrc/build.py)
k=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  SDGR_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --dropin-views 0 --steps 10 > gpurun_out/b_$lib.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/b_$lib.log') if l.startswith('{')][-1])
print('$lib', round(d['value'],1), d['roofline']['kernel_ms_per_step'].get('$k'), round(d['preprocess_sort_roofline']['frac_comp_plane_only'],4))"
done
