set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --steps 50 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
KS_FD_DEDUP=0 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-solve > gpurun_out/bench_nodedup.log 2>&1
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fd_solve|k_kron_level" -s 1 -c 6 -o gpurun_out/prof_c3d python tools/prof_c3.py c3 > gpurun_out/ncu_full.log 2>&1
