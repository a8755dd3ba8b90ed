# round 2: launch list of one 16-view c4 step + ncu --set full of the top kernels
# (from the repo root on the GPU box; each ncu command runs only after the plain run exited 0)
set -e
python profiles/prof_step.py --views 16 > gpurun_out/plain_r2.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r2.csv python profiles/prof_step.py --views 16 > gpurun_out/ncu_l_r2.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_project|k_walk|k_replay|k_segsum|k_splat|k_gather_prim|k_onesweep|k_grad_geometry" -c 12 \
    -o gpurun_out/full_r2 python profiles/prof_step.py --views 16 > gpurun_out/ncu_f_r2.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k "regex:k_replay|k_grad_image|k_count_emit|k_grad_geometry|k_walk" -c 6 \
    -o gpurun_out/full_r2b python profiles/prof_step.py --views 16 > gpurun_out/ncu_f_r2b.log 2>&1
