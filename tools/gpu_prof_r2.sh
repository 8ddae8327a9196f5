#!/bin/bash
# Round-2 captures: launch list of the bench command (c3, no legs), ncu --set full
# of the fused axis-1 stage and of the folded transforms (prof_c3.py), summaries.
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --no-solve > gpurun_out/r2p_bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/r2p_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --no-solve > gpurun_out/r2p_ncu_launch.log 2>&1
python tools/prof_c3.py c3 > gpurun_out/r2p_plain.log 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_fd_axis1" -s 1 -c 1 \
    -o gpurun_out/r2p_ax1 python tools/prof_c3.py c3 > gpurun_out/r2p_ax1.log 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_xfold" -s 4 -c 4 \
    -o gpurun_out/r2p_xf python tools/prof_c3.py c3 > gpurun_out/r2p_xf.log 2>&1
python tools/ncu_summary.py gpurun_out/r2p_ax1.ncu-rep gpurun_out/r2p_ax1_summary.csv >> gpurun_out/r2p_ax1.log 2>&1
python tools/ncu_summary.py gpurun_out/r2p_xf.ncu-rep gpurun_out/r2p_xf_summary.csv >> gpurun_out/r2p_xf.log 2>&1
echo done
