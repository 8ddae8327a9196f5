#!/bin/bash
mkdir -p gpurun_out
python tools/prof_c5.py > gpurun_out/c5prof_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__block_size,launch__grid_size,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv --log-file gpurun_out/c5_launches.csv python tools/prof_c5.py > gpurun_out/c5prof_ncu.log 2>&1
