for o in native morton random; do for lib in libsdgr_old.so libsdgr.so; do SDGR_LIB=$lib SDGR_BENCH_ORDER=$o python bench.py --no-cpu-baseline --no-e2e --dropin-views 0 --steps 10 > gpurun_out/bb.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bb.log') if l.startswith('{')][-1]); k=d['roofline']['kernel_ms_per_step']
print('$o $lib', round(d['value'],1), k['k_splat'], k['k_grad_image'], k['k_count_emit'], k['k_grad_geometry'])"; done; done
