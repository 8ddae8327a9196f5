#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/kron_sweep.py 'KS_KRON3=0' 'KS_KRON_JIT_MINB=2' 'KS_KRON_JIT_MAXT=256' 'KS_KRON_JIT_MAXT=192' 'KS_KRON_JIT_NOSTAGE=1' > gpurun_out/rank3_sweep.log 2>&1
SWEEP_CFG=c5 timeout 900 python tools/kron_sweep.py 'KS_KRON3=0' 'KS_KRON_JIT_MINB=2' 'KS_KRON_JIT_MAXT=256' >> gpurun_out/rank3_sweep.log 2>&1
rm -f gpurun_out/jit_c3.cu; KS_KRON_JIT_DUMP=$PWD/gpurun_out/jit_c3.cu timeout 600 python tools/kron_sweep.py 'KS_KRON3=0' > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none -k regex:"ks_pair" -c 2 --csv --log-file gpurun_out/rank3_launches.csv python tools/prof_c3.py c3 > /dev/null 2>&1
