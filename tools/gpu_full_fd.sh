#!/bin/bash
# full ncu capture of one FD apply's kernels (fold GEMMs + solve) at c3
mkdir -p gpurun_out
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mode_gemm_fold|k_fd_solve" -c 7 -o gpurun_out/prof_fd_fold python tools/prof_c3.py c3 > gpurun_out/ncu_fd_fold.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_fd_fold.log
