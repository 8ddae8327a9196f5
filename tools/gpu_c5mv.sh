#!/bin/bash
mkdir -p gpurun_out
SWEEP_CFG=c5 timeout 1200 python tools/kron_sweep.py 'KS_KRON3=0' 'KS_KRON_JIT_MAXT=256' 'KS_KRON_JIT_MAXT=192' 'KS_KRON_JIT_MAXT=128' 'KS_KRON_JIT_MINB=2' 'KS_KRON_JIT_MAXT=256 KS_KRON_JIT_MINB=2' 'KS_KRON_JIT_NOSTAGE=1' > gpurun_out/c5mv_sweep.log 2>&1
SWEEP_CFG=c3 timeout 1200 python tools/kron_sweep.py 'KS_KRON3=0' 'KS_KRON3=0 KS_KRON_JIT_MAXT=256' 'KS_KRON3=0 KS_KRON_JIT_MAXT=192' 'KS_KRON3=0 KS_KRON_JIT_MINB=2' >> gpurun_out/c5mv_sweep.log 2>&1
