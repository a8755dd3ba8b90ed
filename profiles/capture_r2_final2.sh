# round 2 evidence, second pass (after the splat warp order, the walk claim
# order and the 24-view batches; from the repo root on the GPU box).  Every
# ncu command runs after the plain command it profiles exited 0.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1
python bench.py > gpurun_out/bench_c4.log 2>&1
python bench.py --workload c2 > gpurun_out/bench_c2.log 2>&1
python bench.py --workload c3 > gpurun_out/bench_c3.log 2>&1
python bench.py --scene-order native --no-cpu-baseline --dropin-views 0 > gpurun_out/bench_c4n.log 2>&1
python profiles/timeline.py > gpurun_out/timeline.json 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dropin-views 0 > gpurun_out/b_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_r2.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --dropin-views 0 > gpurun_out/ncu_l.log 2>&1
python profiles/prof_step.py --views 24 > gpurun_out/plain_r2.log 2>&1 && \
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k "regex:k_project|k_walk|k_replay|k_segsum|k_splat|k_gather_prim|k_onesweep|k_grad_geometry|k_grad_image|k_count_emit" \
      -c 14 -o gpurun_out/full_r2h python profiles/prof_step.py --views 24 > gpurun_out/ncu_h.log 2>&1
ls -la gpurun_out
