#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold.py tests/test_gpu_golden.py -q -x > gpurun_out/nat_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/nat_pytest.log
timeout 900 python tools/fd_sweep.py 'KS_FD_NAT=0' 'KS_FD_NAT=1' > gpurun_out/nat_sweep.log 2>&1
SWEEP_CFG=c5s timeout 900 python tools/fd_sweep.py 'KS_FD_NAT=0' 'KS_FD_NAT=1' >> gpurun_out/nat_sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fold|solve" -c 8 --csv \
    --log-file gpurun_out/nat_launches.csv python tools/prof_c3.py c3 > gpurun_out/nat_ncu.log 2>&1
