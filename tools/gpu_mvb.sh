#!/bin/bash
# Row-blocked matvec candidates: parity (forced), timings of all candidates, bench line
mkdir -p gpurun_out
for v in b2 b4; do
  KS_KRON_JIT=$v timeout 900 python -m pytest tests/test_gpu_kron3.py tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/mvb_tests_$v.log 2>&1
  tail -2 gpurun_out/mvb_tests_$v.log
  grep "candidate" gpurun_out/mvb_tests_$v.log | sort | uniq -c | sort -rn | head -5
done
KS_KRON_JIT=log timeout 600 python tools/prof_c3.py c3 2>&1 | grep -E "candidate|ok" | head -20
KS_KRON_JIT=b2 timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --no-extra --no-cpu-baseline > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'P'
import json
d = json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1])
print('fd ms', d['ms_per_step'], 'matvec', d.get('matvec', {}).get('ms'), 'solve', d['solves']['solve_c3']['seconds'])
P
