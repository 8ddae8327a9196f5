#!/bin/bash
mkdir -p gpurun_out
KS_FOLD_CFG=1 timeout 600 python -m pytest tests/test_gpu_fold.py -q -x > gpurun_out/foldcfg_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/foldcfg_pytest.log
timeout 600 python tools/fd_sweep.py KS_FOLD_CFG=0 KS_FOLD_CFG=1 KS_FOLD_CFG=2 KS_FOLD_CFG=0 KS_FOLD_CFG=1 KS_FOLD_CFG=2 > gpurun_out/foldcfg.log 2>&1
