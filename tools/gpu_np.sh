#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold.py tests/test_gpu_golden.py -q -x > gpurun_out/np_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/np_pytest.log
timeout 600 python tools/fd_sweep.py KS_FD_NOPIV=0 KS_FD_NOPIV=1 > gpurun_out/np_sweep.log 2>&1
SWEEP_CFG=c4p3 timeout 600 python tools/fd_sweep.py KS_FD_NOPIV=0 KS_FD_NOPIV=1 >> gpurun_out/np_sweep.log 2>&1
SOLVE_N=3 timeout 300 python tools/solve_timing.py >> gpurun_out/np_sweep.log 2>&1
