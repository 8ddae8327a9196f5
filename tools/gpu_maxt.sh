#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/kron_sweep.py KS_KRON_JIT_MAXT=128 KS_KRON_JIT_MAXT=192 KS_KRON_JIT_MAXT=256 KS_KRON_JIT_MAXT=320 KS_KRON_JIT_MAXT=384 KS_KRON_JIT_MAXT=448 > gpurun_out/maxt.log 2>&1
