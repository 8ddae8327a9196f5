"""Drop-in demonstration on the GPU: the reference's own pcg (compiled from its
sources into oracle/_ref) runs with the B200 operators behind its ApplyFn
callbacks (oracle/integration_demo.cpp, the binding shown in INTEGRATION.md)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "integration_demo")


@pytest.mark.parametrize("args", [(1, 3, 16), (2, 3, 16), (3, 2, 8)])
def test_reference_pcg_with_gpu_operators(gpu, args):
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/integration_demo not built (needs /root/reference at build time)")
    out = subprocess.run([DEMO, *map(str, args)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert all(r["converged"])
    assert abs(r["gpu_callback_iters"] - r["cpu_iters"]) <= 1
    assert abs(r["gpu_device_iters"] - r["cpu_iters"]) <= 1
    assert r["rel_x_callback"] < 1e-7 and r["rel_x_device"] < 1e-7
