#!/bin/bash
mkdir -p gpurun_out
KS_KRON_JIT_ILV=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matvec or kron or pcg_matches" > gpurun_out/ilv_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ilv_pytest.log
timeout 600 python tools/kron_sweep.py KS_KRON_JIT_ILV=0 KS_KRON_JIT_ILV=1 KS_KRON_JIT_ILV=0 KS_KRON_JIT_ILV=1 > gpurun_out/ilv.log 2>&1
SWEEP_CFG=c5 timeout 600 python tools/kron_sweep.py KS_KRON_JIT_ILV=0 KS_KRON_JIT_ILV=1 >> gpurun_out/ilv.log 2>&1
for c in c4p4 c4p5 c4p6; do SWEEP_CFG=$c timeout 600 python tools/fd_sweep.py KS_FD_NOPIV=0 KS_FD_NOPIV=1 >> gpurun_out/ilv.log 2>&1; done
