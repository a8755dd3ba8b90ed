# launch list of a 2-view c4 step + ncu --set full of the preprocess / sort / binning kernels (1 view)
set -e
python profiles/prof_step.py --views 2 > gpurun_out/plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pre.csv python profiles/prof_step.py --views 2 > gpurun_out/ncu1.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_project|k_key32|k_radix|k_onesweep|k_fix_runs|k_emit|k_gather|k_seg_scan|k_tile_ranges|k_make_items|k_key_range|k_scan}" -c ${KCOUNT:-40} -o gpurun_out/pre python profiles/prof_step.py --views 1 > gpurun_out/ncu2.log 2>&1
