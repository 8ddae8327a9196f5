#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_infsup.py tests/test_gpu_rhs.py -q -x > gpurun_out/pcg_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pcg_pytest.log
timeout 900 python tools/solve_timing.py > gpurun_out/pcg_timing.log 2>&1
