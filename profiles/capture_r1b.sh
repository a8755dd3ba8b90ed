# Round-1 capture (repo root, GPU box): launch list of one 2-view step, then
# ncu --set full of each library kernel (1 view; the geometry epilogue as a
# full 8-view batch), then the traffic summary bench.py reads.
set -e
python profiles/prof_step.py --views 2 > gpurun_out/plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r1.csv python profiles/prof_step.py --views 2 > gpurun_out/ncu1.log 2>&1
python profiles/prof_step.py --views 1 > gpurun_out/plain1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k 'regex:k_project|k_walk|k_segsum|k_replay|k_splat$|k_grad_image|k_gather|k_emit|k_onesweep' -c 16 \
    -o gpurun_out/full_r1 python profiles/prof_step.py --views 1 > gpurun_out/ncu2.log 2>&1
python profiles/prof_step.py --views 8 > gpurun_out/plain8.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k 'regex:k_grad_geometry' -c 1 \
    -o gpurun_out/geo_r1 python profiles/prof_step.py --views 8 > gpurun_out/ncu3.log 2>&1
