for l in 8 6 10 12 16 8; do python bench.py --no-cpu-baseline --no-e2e --dropin-views 0 --steps 10 --lanes $l > gpurun_out/bl.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bl.log') if l.startswith('{')][-1]); print('lanes $l', round(d['value'],1))"; done
for gb in 8 12; do python bench.py --no-cpu-baseline --no-e2e --dropin-views 0 --steps 10 --geo-batch $gb > gpurun_out/bl.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bl.log') if l.startswith('{')][-1]); print('geo-batch $gb', round(d['value'],1))"; done
