#!/bin/bash
# axis-1 time-major hand-off: FD parity tests, then c3 / c5 FD apply timing with it off / on
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fold.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_galerkin.py tests/test_gpu_infsup.py -q -x > gpurun_out/tm1_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/tm1_pytest.log
timeout 600 python tools/fd_sweep.py KS_FD_TM1=0 KS_FD_TM1=1 KS_FD_TM1=0 KS_FD_TM1=1 > gpurun_out/tm1_sweep.log 2>&1
SWEEP_CFG=c5 timeout 600 python tools/fd_sweep.py KS_FD_TM1=0 KS_FD_TM1=1 >> gpurun_out/tm1_sweep.log 2>&1
