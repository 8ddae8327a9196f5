mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kron3.py -m gpu -x -q -k generated 2>&1 | tail -15
KS_KRON_JIT=log timeout 600 python tools/prof_c3.py c3 2>&1 | grep -E "candidate|ok"
KS_KRON_JIT=log timeout 600 python tools/prof_c5mv.py 2>&1 | grep -E "candidate|ok"
