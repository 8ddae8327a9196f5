#!/bin/bash
mkdir -p gpurun_out
python tools/prof_c3.py c3 > gpurun_out/pp_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ks_pair" -c 8 \
    -o gpurun_out/prof_pair python tools/prof_c3.py c3 > gpurun_out/pp_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/pp_ncu.log
