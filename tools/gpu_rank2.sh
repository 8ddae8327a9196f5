#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kron3.py -q -x > gpurun_out/rank_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/rank_pytest.log
timeout 900 python tools/solve_timing.py > gpurun_out/rank_solve.log 2>&1
