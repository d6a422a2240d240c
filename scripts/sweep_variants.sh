#!/bin/bash
# fine-kernel layout variants on the C2 bench (prints value / fine ms)
for v in "2 8" "1 8" "1 16" "2 16"; do
  set -- $v
  PINT_TRI_MINB=$1 PINT_TRI_BATCH_CL=$2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err || { echo "minb=$1 cl=$2 FAILED"; tail -3 /tmp/b.err; continue; }
  python -c "import json; d=json.load(open('/tmp/b.json')); print('minb=$1 cl=$2', round(d['value'],1), 'GPt/s step_ms', round(d['ms_per_step'],3), 'fine_ms', round(d['roofline']['fine_kernel_ms'],3), 'delta', d['delta_first_sweep'])"
done
