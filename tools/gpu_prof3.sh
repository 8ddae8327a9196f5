#!/bin/bash
# full ncu capture of the two fused matvec pass pairs (NVRTC "ks_pair")
mkdir -p gpurun_out
python tools/prof_c3.py c3 > gpurun_out/prof3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ks_pair" -c 2 \
    -o gpurun_out/prof3 python tools/prof_c3.py c3 > gpurun_out/prof3_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof3_ncu.log
