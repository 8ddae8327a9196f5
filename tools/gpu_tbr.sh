#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/fd_sweep.py 'KS_FD_TBR=8' 'KS_FD_TBR=16' 'KS_FD_TBR=32' 'KS_FD_TBR=4' > gpurun_out/tbr_sweep.log 2>&1
SWEEP_CFG=c5s timeout 900 python tools/fd_sweep.py 'KS_FD_TBR=8' 'KS_FD_TBR=16' 'KS_FD_TBR=32' >> gpurun_out/tbr_sweep.log 2>&1
timeout 600 python tools/kron_sweep.py 'KS_KRON3=0' 'KS_KRON3=1' >> gpurun_out/tbr_sweep.log 2>&1
