# quick check: GPU parity suite + short bench, per-view stage times (µs)
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/b.json
python -c "import json; d=json.load(open('gpurun_out/b.json')); print(round(d['value'],1), round(d['e2e']['value'],1), {k: round(v*1000/45,1) for k,v in d['stage_ms_per_step'].items()})"
