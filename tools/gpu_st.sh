#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/fd_sweep.py KS_FOLD_ST=0 KS_FOLD_ST=1 KS_FOLD_ST=2 KS_FOLD_ST=0 KS_FOLD_ST=1 > gpurun_out/st.log 2>&1
