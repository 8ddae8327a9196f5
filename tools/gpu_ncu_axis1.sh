#!/bin/bash
mkdir -p gpurun_out
name=axis1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_fd_axis1" -s 1 -c 1 \
    -o /tmp/prof_$name python tools/prof_c3.py c3 > gpurun_out/ncu_$name.log 2>&1
python tools/ncu_summary.py /tmp/prof_$name.ncu-rep gpurun_out/ncu_${name}_summary.csv >> gpurun_out/ncu_$name.log 2>&1
ncu -i /tmp/prof_$name.ncu-rep --page source --csv > gpurun_out/ncu_${name}_source.csv 2>/dev/null
