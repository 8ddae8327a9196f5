#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/jit_c5.cu gpurun_out/jit_c3.cu
KS_KRON_JIT_DUMP=$PWD/gpurun_out/jit_c5.cu SWEEP_CFG=c5 timeout 600 python tools/kron_sweep.py 'KS_KRON3=0' > gpurun_out/dump.log 2>&1
KS_KRON_JIT_DUMP=$PWD/gpurun_out/jit_c3.cu SWEEP_CFG=c3 timeout 600 python tools/kron_sweep.py 'KS_KRON3=0' >> gpurun_out/dump.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"ks_pair" -c 2 -o gpurun_out/prof_c5pair python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2311_18461_b200 as ks
prob = ks.SpaceTimeProblem.uniform(3, 4, 128, 128)
A = ks.assemble_system_operator(prob)
n = prob.N_dof
x = ks.DeviceVector.from_host(np.ones(n, complex)); y = ks.DeviceVector(n)
A.apply(x, y); ks.lib().ks_synchronize()
" >> gpurun_out/dump.log 2>&1
