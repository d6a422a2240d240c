#!/bin/bash
# Round-2 evidence in one GPU call (outputs under gpurun_out/r2ev_*): smoke,
# the ncu launch list of a short bench run (after the same command ran clean
# without ncu) and full captures of the dominant kernels: the C2 fine kernel,
# the TMA 3-D stencil at C4, the 2-D stencil at C3.
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ev_smoke.log 2>&1; tail -1 gpurun_out/r2ev_smoke.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-time-to-tol --no-configs"
timeout 600 $B > gpurun_out/r2ev_bench_short.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2ev_launches.csv $B > gpurun_out/r2ev_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tri1d_batch_kernel -c 1 \
  -o gpurun_out/r2ev_fine -f python scripts/profile_c2.py fine > gpurun_out/r2ev_ncu_fine.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fe3d_tile -c 1 \
  -o gpurun_out/r2ev_fe3d -f python scripts/profile_nd.py c4_f32 16 3 > gpurun_out/r2ev_ncu_fe3d.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fe2d_wave -c 1 \
  -o gpurun_out/r2ev_fe2d -f python scripts/profile_nd.py c3_f64 32 8 > gpurun_out/r2ev_ncu_fe2d.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tri1d_sweep_kernel -c 1 \
  -o gpurun_out/r2ev_sweep -f python scripts/profile_c2.py sweep > gpurun_out/r2ev_ncu_sweep.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:xform_tc -c 2 \
  -o gpurun_out/r2ev_xform -f python scripts/profile_coarse.py c4_f32 2 > gpurun_out/r2ev_ncu_xform.log 2>&1
# summaries on the box (the reports are too large to bring back all at once)
python scripts/ncu_summary.py gpurun_out/r2ev_*.ncu-rep --launches gpurun_out/r2ev_launches.csv \
  > gpurun_out/r2ev_summary.txt 2>&1
for r in gpurun_out/r2ev_*.ncu-rep; do
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}_details.csv" 2>/dev/null
done
rm -f gpurun_out/r2ev_*.ncu-rep
ls -la gpurun_out | grep r2ev
