python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_shard.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline --no-solve > gpurun_out/bench.log 2>&1
KS_GEMM_V2=1 python bench.py --steps 20 --no-cpu-baseline --no-solve > gpurun_out/bench_v2.log 2>&1
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mode_gemm" -c 3 -o gpurun_out/prof_gemm3 python tools/prof_c3.py c3 > gpurun_out/ncu_gemm3.log 2>&1
