#!/bin/bash
# Debug library with per-phase clock64 stamps (scripts/phase_timing.py).
set -e
cd "$(dirname "$0")/.."
C=paper_2110_10762_b200/csrc
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -DPINT_PHASE_TIMING \
  $C/abi.cu $C/tri1d.cu $C/correct.cu $C/stencil.cu $C/stencil_wave.cu $C/cg.cu $C/spectral.cu \
  -o scripts/libpint_timing.so -lcudart
