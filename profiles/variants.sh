# A/B of library variants built with SDGR_LIB_NAME (see csrc/build.py):
#   bash profiles/variants.sh libsdgr.so libsdgr_x.so ...
# prints views/s, e2e and the single-stream per-kernel ms/step of each.
for lib in "$@"; do
  SDGR_LIB=$lib python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/v.json
  python -c "
import json; d=json.load(open('gpurun_out/v.json')); r=d['roofline']
print('$lib', round(d['value'],1), round(d['e2e']['value'],1), r['kernel_ms_per_step'])"
done
