#!/bin/bash
# fold transform round: GPU tests, c3 + c5 bench, quick ncu launch list of c3 FD + matvec
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --no-solve --steps 20 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_c5.log 2>&1
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/quick.csv python tools/prof_c3.py c3 > gpurun_out/ncu_quick.log 2>&1
