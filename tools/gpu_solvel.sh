#!/bin/bash
mkdir -p gpurun_out
SOLVE_N=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/solve_launches2.csv python tools/solve_timing.py > gpurun_out/psolve2.log 2>&1
