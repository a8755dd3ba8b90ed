# ncu --set full of the batched preprocessing kernels (one 8-view batch), from the repo root on the GPU box
set -e
ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_project|k_key|k_onesweep|k_fix_runs|k_emit|k_gather|k_scan|k_make_items|k_range_init}" -c ${KCOUNT:-40} -o gpurun_out/batch python profiles/prof_step.py --views 8 > gpurun_out/ncu_b.log 2>&1
