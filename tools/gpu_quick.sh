#!/bin/bash
# Quick check after an FD kernel change: the FD parity tests, then the c3 bench line without legs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fold.py tests/test_gpu_golden.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/quick_tests.log 2>&1
tail -3 gpurun_out/quick_tests.log
timeout 600 python bench.py --no-extra --no-cpu-baseline --no-solve > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'P'
import json
d = json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1])
print('fd ms', d['ms_per_step'], 'components', json.dumps(d['fd_apply']['components_ms_per_apply']), 'roofline', d['roofline']['frac'], 'matvec', d.get('matvec', {}).get('ms'))
P
