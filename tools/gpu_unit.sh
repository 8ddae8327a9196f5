#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kron3.py tests/test_gpu_rhs.py -q -x > gpurun_out/unit_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/unit_pytest.log
timeout 600 python tools/kron_sweep.py KS_KRON_JIT_UNIT=0 KS_KRON_JIT_UNIT=1 KS_KRON_JIT_UNIT=0 KS_KRON_JIT_UNIT=1 > gpurun_out/unit.log 2>&1
SWEEP_CFG=c5 timeout 600 python tools/kron_sweep.py KS_KRON_JIT_UNIT=0 KS_KRON_JIT_UNIT=1 >> gpurun_out/unit.log 2>&1
rm -f gpurun_out/jit_src.cu; KS_KRON_JIT_DUMP=gpurun_out/jit_src.cu timeout 300 python tools/kron_sweep.py KS_KRON_JIT_UNIT=1 >> gpurun_out/unit.log 2>&1
