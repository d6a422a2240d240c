#!/bin/bash
# Full ncu capture (with source page) of the fused coarse sweep at C2.
set -e
tag=${1:-sweep}
python scripts/profile_c2.py sweep > gpurun_out/${tag}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tri1d_sweep_kernel -c 1 \
  -o gpurun_out/${tag} -f python scripts/profile_c2.py sweep > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv > gpurun_out/${tag}_source.csv 2>/dev/null || true
rm -f gpurun_out/${tag}.ncu-rep
python scripts/sweep_time.py
