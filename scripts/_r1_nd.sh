set -x
mkdir -p gpurun_out
timeout 900 python scripts/bench_configs.py all --tol > gpurun_out/nd_configs2.jsonl 2> gpurun_out/nd_configs2.err
python scripts/profile_nd.py c4_f32 4 4 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:fe3d_tile -c 1 -o gpurun_out/prof_fe3d_v8 -f python scripts/profile_nd.py c4_f32 4 4 > gpurun_out/ncu_fe3d_v8.log 2>&1
python scripts/profile_nd.py c3_f64 32 8 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:fe2d_wave -c 1 -o gpurun_out/prof_fe2d_full -f python scripts/profile_nd.py c3_f64 32 8 > gpurun_out/ncu_fe2d_full.log 2>&1
cat gpurun_out/nd_configs2.jsonl; tail -3 gpurun_out/nd_configs2.err
