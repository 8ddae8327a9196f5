#!/bin/bash
# fused axis-1/2 transform: parity tests, timing vs the unfused passes, launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fold.py -q -x > gpurun_out/f12_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/f12_pytest.log
timeout 600 python tools/fd_sweep.py 'KS_FD_FUSE12=0' 'KS_FD_FUSE12=1' > gpurun_out/f12_sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum --clock-control none -c 40 --csv \
    --log-file gpurun_out/f12_launches.csv python tools/prof_c3.py c3 > gpurun_out/f12_ncu.log 2>&1
