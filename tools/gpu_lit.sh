#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_rhs.py -q -x > gpurun_out/lit_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/lit_pytest.log
timeout 900 python tools/kron_sweep.py 'KS_KRON3=0' > gpurun_out/lit_sweep.log 2>&1
SWEEP_CFG=c5 timeout 900 python tools/kron_sweep.py 'KS_KRON3=0' >> gpurun_out/lit_sweep.log 2>&1
timeout 900 python tools/solve_timing.py > gpurun_out/lit_solve.log 2>&1
