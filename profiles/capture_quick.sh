# launch list + ncu --set full of the comp-plane kernels (1 view), from the repo root on the GPU box
set -e
python profiles/prof_step.py --views 2 > gpurun_out/plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python profiles/prof_step.py --views 2 > gpurun_out/ncu1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_segsum|k_walk|k_replay}" -c ${KCOUNT:-4} -o gpurun_out/q python profiles/prof_step.py --views 1 > gpurun_out/ncu2.log 2>&1
