# Round-1 (batched preprocessing) capture, repo root on the GPU box:
#  1. launch list of the bench command itself (first 400 kernels: warm-up step),
#  2. launch list of one full 16-view batch step (prof_step.py),
#  3. ncu --set full of every library kernel of that batch step,
#  4. the traffic summary bench.py reads (profiles/ncu_traffic.json).
set -e
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu0.log 2>&1
python profiles/prof_step.py --views 16 > gpurun_out/plain16.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r1c.csv python profiles/prof_step.py --views 16 > gpurun_out/ncu1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k 'regex:k_project$|k_key|k_onesweep|k_fix_runs|k_count_emit|k_gather|k_make_items|k_segsum|k_walk|k_replay|k_splat$|k_grad_image|k_grad_geometry|k_seg_scan|k_reduce' \
    -c 22 -o gpurun_out/full_r1c python profiles/prof_step.py --views 16 > gpurun_out/ncu2.log 2>&1
python profiles/make_traffic.py profiles/ncu_traffic.json gpurun_out/full_r1c.ncu-rep
