#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold.py tests/test_gpu_golden.py tests/test_gpu_shard.py tests/test_galerkin.py -q -x > gpurun_out/np_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/np_pytest.log
timeout 600 python tools/fd_sweep.py KS_FD_NOPIV=0 KS_FD_NOPIV=1 > gpurun_out/np_sweep.log 2>&1
for c in c4p2 c4p3 c2; do SWEEP_CFG=$c timeout 600 python tools/fd_sweep.py KS_FD_NOPIV=0 KS_FD_NOPIV=1 >> gpurun_out/np_sweep.log 2>&1; done
