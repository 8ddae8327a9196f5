#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_parity.py tests/test_gpu_rhs.py tests/test_galerkin.py tests/test_gpu_shard.py -q -x > gpurun_out/rank_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/rank_pytest.log
KS_KRON3=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x > gpurun_out/rank_pytest2.log 2>&1
echo "rc=$?" >> gpurun_out/rank_pytest2.log
timeout 600 python tools/kron_sweep.py 'KS_KRON3=0 KS_KRON_RANK=0' 'KS_KRON3=0' 'KS_KRON3=1' > gpurun_out/rank_sweep.log 2>&1
SWEEP_CFG=c5 timeout 600 python tools/kron_sweep.py 'KS_KRON_RANK=0' 'KS_KRON3=0' >> gpurun_out/rank_sweep.log 2>&1
SWEEP_CFG=c2 timeout 600 python tools/kron_sweep.py 'KS_KRON_RANK=0' 'KS_KRON3=0' >> gpurun_out/rank_sweep.log 2>&1
