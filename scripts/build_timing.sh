#!/bin/bash
# Debug library with per-phase clock64 stamps (scripts/phase_timing.py).
set -e
cd "$(dirname "$0")/.."
C=paper_2110_10762_b200/csrc
B=$C/_build
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  --expt-relaxed-constexpr -DPINT_PHASE_TIMING -c $C/tri1d.cu -o /tmp/tri1d_timing.o
objs=""
for f in abi async_rt correct stencil stencil_wave stencil3d cg spectral tc_xform mailbox; do objs="$objs $B/$f.o"; done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC $objs /tmp/tri1d_timing.o \
  -o scripts/libpint_timing.so -lcudart
