#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold.py tests/test_gpu_golden.py -q -x > gpurun_out/nat_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/nat_pytest.log
timeout 900 python tools/fd_sweep.py 'KS_FD_NAT=0' 'KS_FD_NAT=1' > gpurun_out/nat_sweep.log 2>&1
SWEEP_CFG=c5s timeout 900 python tools/fd_sweep.py 'KS_FD_NAT=0' >> gpurun_out/nat_sweep.log 2>&1
