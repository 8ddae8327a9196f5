#!/bin/bash
# c2 (d=2, 279 K DOF): parity of the small-grid kernels, solve time, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold.py tests/test_gpu_golden.py tests/test_gpu_rhs.py -q -x > gpurun_out/c2_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c2_pytest.log
python tools/prof_c2.py > gpurun_out/c2_plain.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/c2_launches.csv python tools/prof_c2.py > gpurun_out/c2_ncu.log 2>&1
