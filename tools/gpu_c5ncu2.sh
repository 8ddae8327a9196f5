#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_xfold" -s 7 -c 1 \
    -o /tmp/prof_c5xf python tools/prof_c5.py > gpurun_out/ncu_c5xf.log 2>&1
python tools/ncu_summary.py /tmp/prof_c5xf.ncu-rep gpurun_out/ncu_c5xf_summary.csv >> gpurun_out/ncu_c5xf.log 2>&1
ncu -i /tmp/prof_c5xf.ncu-rep --page source --csv > gpurun_out/ncu_c5xf_source.csv 2>/dev/null
