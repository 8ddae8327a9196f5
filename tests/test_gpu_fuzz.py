"""Random problem shapes (d, degree, elements in space and time) through the default kernel selection
and with the generated tile kernel and the position-ordered d = 2 plan forced: system matvec and FD
application against the oracle, <= 1e-10 relative (tools/fuzz_shapes.py; the environment switches are
read per process, hence the subprocesses)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env,seed", [({}, 11), ({"KS_KRON_JIT": "tile", "KS_FD_XFOLD": "1"}, 12),
                                      ({"KS_KRON_JIT": "b2", "KS_FD_DEDUP": "1"}, 13)])
def test_random_shapes_match_oracle(env, seed):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_shapes.py"), str(seed), "7"],
                         env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-1500:], out.stderr[-1500:])
    assert float(out.stdout.strip().split()[-1]) <= 1e-10
