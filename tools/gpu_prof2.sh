#!/bin/bash
# full ncu captures: fused axis-1/2 transform (fwd + inv) and the two fused matvec pass pairs
mkdir -p gpurun_out
export KS_FD_FUSE12=1
python tools/prof_c3.py c3 > gpurun_out/prof2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fold12|ks_pair" -c 4 \
    -o gpurun_out/prof2 python tools/prof_c3.py c3 > gpurun_out/prof2_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/prof2_ncu.log
