#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/fd_sweep.py KS_FOLD_DRY=0 KS_FOLD_DRY=1 KS_FOLD_DRY=2 KS_FOLD_DRY=3 > gpurun_out/dry.log 2>&1
