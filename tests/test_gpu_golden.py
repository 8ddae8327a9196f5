"""GPU parity against golden vectors produced by the reference's own code
(tests/golden/make_golden.py): inputs are the reference's setup products,
outputs compared at the north_star tolerance (1e-10 relative per application,
PCG iterations +-1)."""
import numpy as np
import pytest

from golden_io import cases, tw_cases, load, ids
from helpers import rel, maxrel

pytestmark = pytest.mark.gpu


def _gpu_ops(ks, oracle, g):
    P = ks.FDPreconditioner.from_arrays(g["dims"], 1.0, g["p"], g["U"], g["lam"], g["Lt"],
                                        g["Mt"], g["Wt"])
    A = ks.KroneckerOperator(g["dims"])
    for c, fs, bw in oracle.system_terms(g, g["d"], 1.0):
        A.add_term(c, [ks.Banded(g["dims"][k], bw[k], f) for k, f in enumerate(fs)])
    return P, A


@pytest.mark.parametrize("path", cases(), ids=ids(cases()))
def test_gpu_vs_reference_golden(gpu, oracle, path):
    g = load(path)
    P, A = _gpu_ops(gpu, oracle, g)
    r = g["r"]
    z = P.apply(r)
    for key in ("z", "z_avx2"):
        assert rel(z, g[key]) <= 1e-10 and maxrel(z, g[key]) <= 1e-10
    y = A.apply(r)
    for key in ("y", "y_avx2"):
        assert rel(y, g[key]) <= 1e-10 and maxrel(y, g[key]) <= 1e-10
    assert np.array_equal(P.eigenvalues(), g["lam_composite"])
    ab, piv = P.block(int(g["block_index"]), g["p"])
    assert np.array_equal(piv, g["block_piv"])
    assert maxrel(ab, g["block_ab"]) < 1e-13
    s = gpu.pcg(A, P, r, gpu.PcgOptions(1e-8, 200))
    assert s.converged
    assert abs(s.iterations - int(g["pcg_iters"])) <= 1
    assert rel(s.x, g["pcg_x"]) < 1e-7


@pytest.mark.parametrize("path", tw_cases(), ids=ids(tw_cases()))
def test_gpu_table2_traveling_wave(gpu, oracle, path):
    g = load(path)
    g["d"] = 2
    P, A = _gpu_ops(gpu, oracle, g)
    s = gpu.pcg(A, P, g["b"], gpu.PcgOptions(1e-8, 200))
    assert s.converged
    assert abs(s.iterations - int(g["pcg_iters"])) <= 1
    assert abs(s.iterations - {2: 7, 3: 9, 4: 10}[g["p"]]) <= 2


FC = [p for p in cases() if "case_fc_" in p]


@pytest.mark.parametrize("path", FC, ids=ids(FC))
def test_gpu_final_condition_own_setup(gpu, oracle, path):
    """Final-condition trial space (time basis drops its last function,
    assembly.hpp:59-62) built by libks's own host setup:
    same FD / matvec / PCG kernels, results against the reference's golden
    outputs at the north_star tolerance."""
    g = load(path)
    d, p = g["d"], g["p"]
    prob = gpu.SpaceTimeProblem.uniform(d, p, g["dims"][1] + 2 - p, g["dims"][0] + 1 - p, trial="final")
    assert prob.reduced_dims() == g["dims"]
    P = gpu.FDPreconditioner(prob)
    A = gpu.assemble_system_operator(prob)
    r = g["r"]
    assert rel(P.apply(r), g["z"]) <= 1e-10
    assert rel(A.apply(r), g["y"]) <= 1e-10
    s = gpu.pcg(A, P, r, gpu.PcgOptions(1e-8, 200))
    assert s.converged and abs(s.iterations - int(g["pcg_iters"])) <= 1
