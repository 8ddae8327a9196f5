#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold.py tests/test_gpu_infsup.py tests/test_gpu_integration.py -q -x > gpurun_out/fdot_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/fdot_pytest.log
SOLVE_N=4 KS_PCG_FUSEDOT=0 timeout 300 python tools/solve_timing.py > gpurun_out/fdot.log 2>&1
echo "--- fused" >> gpurun_out/fdot.log
SOLVE_N=4 timeout 300 python tools/solve_timing.py >> gpurun_out/fdot.log 2>&1
