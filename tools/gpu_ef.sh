#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fold.py -q -x -k "pair or pivot or handoff" > gpurun_out/ef_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ef_pytest.log
timeout 600 python tools/fd_sweep.py KS_FD_TM1=1 "KS_LIB_PATH=$PWD/exp/libks_noef.so" KS_FD_TM1=1 "KS_LIB_PATH=$PWD/exp/libks_noef.so" > gpurun_out/ef.log 2>&1
SWEEP_CFG=c5 timeout 600 python tools/fd_sweep.py KS_FD_TM1=1 "KS_LIB_PATH=$PWD/exp/libks_noef.so" >> gpurun_out/ef.log 2>&1
