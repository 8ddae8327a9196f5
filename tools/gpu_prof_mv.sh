#!/bin/bash
# ncu: full capture of the fused matvec pairs (c3) and a launch list of one c3 solve
mkdir -p gpurun_out
python tools/prof_c3.py c3 > gpurun_out/pmv_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ks_pair" -c 16 \
    -o gpurun_out/prof_mv python tools/prof_c3.py c3 > gpurun_out/pmv_ncu.log 2>&1
SOLVE_N=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/solve_launches.csv python tools/solve_timing.py > gpurun_out/psolve.log 2>&1
echo done >> gpurun_out/pmv_ncu.log
