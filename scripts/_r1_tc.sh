mkdir -p gpurun_out
python scripts/profile_coarse.py c4_f32 2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/coarse_c4_tc_launches.csv python scripts/profile_coarse.py c4_f32 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:xform_tc -c 1 -o gpurun_out/prof_xform_tc -f python scripts/profile_coarse.py c4_f32 1 > gpurun_out/ncu_xform_tc.log 2>&1
tail -1 gpurun_out/ncu_xform_tc.log
timeout 900 python scripts/bench_configs.py c4 --tol > gpurun_out/nd_c4_tc.jsonl 2>&1; cut -c1-400 gpurun_out/nd_c4_tc.jsonl
timeout 900 python scripts/c5_lean.py 1e-5 > gpurun_out/c5_lean_tc.json 2>&1; cut -c1-400 gpurun_out/c5_lean_tc.json
