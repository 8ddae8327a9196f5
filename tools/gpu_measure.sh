#!/bin/bash
# Round-1 part-3 measurement pass: GPU tests, default bench, c5 bench, matvec sweep,
# ncu launch list of the bench command, full capture of the dominant kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "rc=$?" >> gpurun_out/bench.log

timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_c5.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu_launch.log 2>&1
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mode_gemm_fold|k_fd_solve_pair|ks_pair" -c 12 \
    -o gpurun_out/prof_top python tools/prof_c3.py c3 > gpurun_out/ncu_top.log 2>&1
echo "done" >> gpurun_out/ncu_top.log
