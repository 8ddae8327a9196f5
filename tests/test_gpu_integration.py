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


def test_async_host_pipeline_matches_blocking(gpu, oracle):
    """ks_fd_apply with host pointers on a user stream (pipelined copies and
    two staging buffers) gives the same results as the blocking call."""
    import numpy as np
    from helpers import setup_arrays
    a = setup_arrays(gpu, 3, 2, 10, 8)
    P = gpu.FDPreconditioner.from_arrays(a["dims"], a["nu"], a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    n = P.vec_size()
    rs = [oracle.random_vec(n, s) for s in range(5)]
    ref = [P.apply(r) for r in rs]
    st = gpu.Stream()
    outs = [np.empty(n, dtype=np.complex128) for _ in rs]
    for r, z in zip(rs, outs):
        P.apply(r, z, stream=st)
    st.synchronize()
    for z, zr in zip(outs, ref):
        assert np.array_equal(z, zr)
