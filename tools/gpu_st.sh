#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/fd_sweep.py KS_FD_TM1=1 KS_FD_TM1=1 > gpurun_out/st.log 2>&1
SWEEP_CFG=c5 timeout 600 python tools/fd_sweep.py KS_FD_TM1=1 >> gpurun_out/st.log 2>&1
SWEEP_CFG=c4p3 timeout 600 python tools/fd_sweep.py KS_FD_TM1=1 >> gpurun_out/st.log 2>&1
