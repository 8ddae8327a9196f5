#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "device_path or alias or fd_apply_matches" > gpurun_out/e2e_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/e2e_pytest.log
timeout 600 python bench.py --no-solve --no-cpu-baseline > gpurun_out/e2e_bench.log 2>&1
