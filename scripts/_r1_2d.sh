mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nd.py -x -q -k "explicit or reduced" > gpurun_out/pytest_2d.log 2>&1; tail -2 gpurun_out/pytest_2d.log
timeout 600 python scripts/bench_configs.py c3 > gpurun_out/nd_c3.jsonl 2>&1; cut -c1-220 gpurun_out/nd_c3.jsonl
