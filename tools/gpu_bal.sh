#!/bin/bash
# Fold-transform wave balancing (KS_FOLD_BAL): GPU tests on the default, then
# FD apply time with balancing off / on at c3, c2, c4 p=3, c5-shaped p=4, c5.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in c3 c2 c4p3 c5s c3 c5; do
  SWEEP_CFG=$c timeout 900 python tools/fd_sweep.py 'KS_FOLD_BAL=0' 'KS_FOLD_BAL=1' 'KS_FOLD_BAL=0' 'KS_FOLD_BAL=1' >> gpurun_out/bal_sweep.log 2>&1
  echo "cfg $c done" >> gpurun_out/bal_sweep.log
done
