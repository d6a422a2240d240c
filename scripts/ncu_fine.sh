#!/bin/bash
# One full ncu capture of the C2 fine batch kernel (after the plain run exits 0).
# usage: scripts/ncu_fine.sh <tag> [env...]
set -e
tag=$1; shift || true
python scripts/fine_ab.py BASE=1 > gpurun_out/fine_${tag}.jsonl
ncu --set full --clock-control none --import-source on -k regex:tri1d_batch -s 1 -c 1 \
  -o gpurun_out/fine_${tag} -f python scripts/fine_ab.py BASE=1 > gpurun_out/fine_${tag}_ncu.log 2>&1
ncu -i gpurun_out/fine_${tag}.ncu-rep --page raw --csv > gpurun_out/fine_${tag}_raw.csv
ncu -i gpurun_out/fine_${tag}.ncu-rep --page source --csv > gpurun_out/fine_${tag}_source.csv 2>/dev/null || true
cat gpurun_out/fine_${tag}.jsonl
