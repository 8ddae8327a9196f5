#!/bin/bash
# matvec ring-depth / block-shape sweep (c3, c5)
mkdir -p gpurun_out
V="KS_KRON_JIT_D=4 KS_KRON_JIT_D=6 KS_KRON_JIT_D=8 KS_KRON_JIT_D=10"
timeout 600 python tools/kron_sweep.py $V 'KS_KRON_JIT_D=8 KS_KRON_JIT_MAXT=384' 'KS_KRON_JIT_D=8 KS_KRON_JIT_MAXT=192' 'KS_KRON_JIT_D=8 KS_KRON_JIT_MAXT=128' 'KS_KRON_JIT_D=4 KS_KRON_JIT_MAXT=384' 'KS_KRON_JIT_D=4 KS_KRON_JIT_MAXT=128' > gpurun_out/ring_sweep.log 2>&1
SWEEP_CFG=c5 timeout 900 python tools/kron_sweep.py KS_KRON_JIT_D=4 KS_KRON_JIT_D=8 >> gpurun_out/ring_sweep.log 2>&1
