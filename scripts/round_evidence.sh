#!/bin/bash
# One GPU call that refreshes the round's evidence under gpurun_out/:
# GPU tests, smoke, the default bench line, the ncu launch list of one bench
# run and full captures of the dominant kernels (each after its command ran
# clean), the 2-D/3-D configurations.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-time-to-tol > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-time-to-tol \
    > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tri1d_batch_kernel -c 1 \
  -o gpurun_out/prof_fine -f python scripts/profile_c2.py fine > gpurun_out/ncu_fine.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fe2d_wave -c 1 \
  -o gpurun_out/prof_fe2d -f python scripts/profile_nd.py c3_f64 32 8 > gpurun_out/ncu_fe2d.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fe3d_tile -c 1 \
  -o gpurun_out/prof_fe3d -f python scripts/profile_nd.py c4_f32 16 3 > gpurun_out/ncu_fe3d.log 2>&1
timeout 900 python scripts/bench_configs.py all --tol > gpurun_out/nd_configs.jsonl 2>&1
timeout 300 python scripts/c1_time.py > gpurun_out/c1_time.json 2>&1
timeout 600 python scripts/c5_lean.py 1e-5 > gpurun_out/c5_lean.json 2>&1
timeout 900 python scripts/async_nd.py 1e-5 > gpurun_out/async_nd_c4.jsonl 2>&1
ls -la gpurun_out | head -40
