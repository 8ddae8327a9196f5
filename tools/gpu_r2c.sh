#!/bin/bash
# round-2c pass: GPU tests, smoke, bench (all legs), reference arm, c5 matvec candidate timings
mkdir -p gpurun_out
KS_KRON_JIT=log timeout 900 python tools/prof_c5.py 2>&1 | grep -E "candidate|ok" > gpurun_out/c5_candidates.log
cat gpurun_out/c5_candidates.log
if [ -z "$SKIP_TESTS" ]; then
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "rc=$?" >> gpurun_out/bench.log
tail -c 1500 gpurun_out/bench.log
if [ -z "$SKIP_REF" ]; then
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
tail -c 600 gpurun_out/bench_ref.log
fi
