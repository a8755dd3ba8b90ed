# Capture recipe for the round-1 profiles (run from the repo root on the GPU box).
set -e
python bench.py > gpurun_out/bench_r1_full.log 2>&1
python profiles/prof_step.py --views 2 > gpurun_out/plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1g.csv python profiles/prof_step.py --views 2 > gpurun_out/ncu1.log 2>&1
python profiles/prof_step.py --views 1 > gpurun_out/plain1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k 'regex:k_project|k_walk|k_segsum|k_replay|k_grad_geometry|k_splat$|k_gather|k_emit' -c 12 -o gpurun_out/full_r1 python profiles/prof_step.py --views 1 > gpurun_out/ncu2.log 2>&1
python bench.py --impl reference > gpurun_out/bench_r1_ref.log 2>&1
