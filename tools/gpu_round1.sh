set -x
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
KS_GEMM=dfma python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_dfma.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu.log 2>&1
