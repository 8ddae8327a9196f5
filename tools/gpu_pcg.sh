#!/bin/bash
# PCG changes: parity tests, c3 solve timing with the deferred x update off / on, matvec timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold.py -q -x > gpurun_out/pcg_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pcg_pytest.log
SOLVE_N=4 KS_PCG_XDEFER=0 timeout 300 python tools/solve_timing.py > gpurun_out/pcg_solve.log 2>&1
echo "--- xdefer" >> gpurun_out/pcg_solve.log
SOLVE_N=4 timeout 300 python tools/solve_timing.py >> gpurun_out/pcg_solve.log 2>&1
timeout 300 python tools/kron_sweep.py KS_KRON_JIT=1 KS_KRON_JIT=1 >> gpurun_out/pcg_solve.log 2>&1
