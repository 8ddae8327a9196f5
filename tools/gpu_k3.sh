#!/bin/bash
# two-launch d=3 matvec: parity tests, timing vs the pass-pair plan, launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_parity.py -q > gpurun_out/k3_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/k3_pytest.log
timeout 600 python tools/kron_sweep.py 'KS_KRON3=0' 'KS_KRON3=1' 'KS_KRON3_TX=2' 'KS_KRON3_TX=3' 'KS_KRON3_TX=4' 'KS_KRON3_TX=6' > gpurun_out/k3_sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:"ks_k3|k_axis3" -c 2 --csv \
    --log-file gpurun_out/k3_launches.csv python tools/prof_c3.py c3 > gpurun_out/k3_ncu.log 2>&1
