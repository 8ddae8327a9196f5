set -x
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mode_gemm|k_fd_solve|k_kron_level" -s 1 -c 9 -o gpurun_out/prof_c3 python tools/prof_c3.py c3 > gpurun_out/ncu_full.log 2>&1
