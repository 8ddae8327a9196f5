#!/bin/bash
# quick check incl. the c5 leg: FD parity tests, c3 bench line with legs (no CPU baseline / solves)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fold.py tests/test_gpu_golden.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/quick_tests.log 2>&1
tail -3 gpurun_out/quick_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'P'
import json
d = json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1])
print('fd ms', d['ms_per_step'], 'components', json.dumps(d['fd_apply']['components_ms_per_apply']), 'roofline', d['roofline']['frac'], 'matvec', d.get('matvec', {}).get('ms'))
print('solve', d['solves'])
c5 = d['legs']['c5']
print('c5 fd', c5['fd_apply']['ms'], 'transforms', c5['fd_apply']['transform_ms_per_apply'], 'matvec', c5['matvec']['ms'], 'solve', c5['solve']['seconds'])
P
