#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/nat_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/nat_pytest.log
timeout 900 python tools/fd_sweep.py 'KS_FD_NAT=0' 'KS_FD_NAT=1' > gpurun_out/nat_sweep.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_fd_solve_nat" -c 1 -o gpurun_out/prof_nat python tools/prof_c3.py c3 > gpurun_out/nat_ncu.log 2>&1
