#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/c4_sweep.py > gpurun_out/c4_sweep.jsonl 2> gpurun_out/c4_sweep.err
timeout 300 python tools/fd_sweep.py 'KS_FD_RING=4' > gpurun_out/c4_fd.log 2>&1
SWEEP_CFG=c4p2 timeout 300 python tools/fd_sweep.py 'KS_FD_RING=4' >> gpurun_out/c4_fd.log 2>&1
SWEEP_CFG=c4p3 timeout 300 python tools/fd_sweep.py 'KS_FD_RING=4' >> gpurun_out/c4_fd.log 2>&1
