#!/bin/bash
# PCG with graph-replayed iteration phases: parity tests, c3 / c2 solve timings (graphs on / off)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_rhs.py tests/test_gpu_integration.py tests/test_gpu_infsup.py -q -x > gpurun_out/graph_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/graph_pytest.log
timeout 900 python tools/solve_timing.py > gpurun_out/graph_solve.log 2>&1
KS_PCG_GRAPH=0 timeout 900 python tools/solve_timing.py >> gpurun_out/graph_solve.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/graph_bench.log 2>&1
KS_PCG_GRAPH=0 timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/graph_bench0.log 2>&1
