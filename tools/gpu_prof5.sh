#!/bin/bash
mkdir -p gpurun_out
python tools/prof_c3.py c3 > gpurun_out/prof5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ks_k3" -c 1 \
    -o gpurun_out/prof5 python tools/prof_c3.py c3 > gpurun_out/prof5_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof5_ncu.log
