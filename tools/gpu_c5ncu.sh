#!/bin/bash
# c5 (n = 130, p = 4): launch list of two FD applications + matvecs, and one
# full capture of a k_xfold launch (source page exported); DFMA latency micro.
mkdir -p gpurun_out
nvcc -O2 -arch=sm_100a -o /tmp/fp64_lat tools/micro/fp64_latency.cu && /tmp/fp64_lat > gpurun_out/fp64_latency.json 2>&1
bash tools/gpu_c5prof.sh
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_xfold" -s 7 -c 1 \
    -o /tmp/prof_c5xf python tools/prof_c5.py > gpurun_out/ncu_c5xf.log 2>&1
python tools/ncu_summary.py /tmp/prof_c5xf.ncu-rep gpurun_out/ncu_c5xf_summary.csv >> gpurun_out/ncu_c5xf.log 2>&1
ncu -i /tmp/prof_c5xf.ncu-rep --page raw --csv > gpurun_out/ncu_c5xf_raw.csv 2>/dev/null
ncu -i /tmp/prof_c5xf.ncu-rep --page source --csv > gpurun_out/ncu_c5xf_source.csv 2>/dev/null
ncu -i /tmp/prof_c5xf.ncu-rep --page details > gpurun_out/ncu_c5xf_details.txt 2>/dev/null
