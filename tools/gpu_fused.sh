python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
KS_FD_FUSED=0 python bench.py --steps 20 --no-cpu-baseline --no-solve > gpurun_out/bench_nofuse.log 2>&1
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fd_fused|k_mode_gemm" -c 3 -o gpurun_out/prof_fused python tools/prof_c3.py c3 > gpurun_out/ncu_fused.log 2>&1
