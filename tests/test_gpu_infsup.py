"""Inf-sup constants (infsup_constant, experiments.cpp:185-232; SURVEY 8(f)
rank 3) from Lanczos (krylov.cpp:116-179) over the GPU operators: system and
space-time mass operators, FD-PCG inner solves (least squares) and the
Galerkin fast solver with its adjoint. The spaces are small enough that the
Krylov space is exhausted, so the reference's values (tests/golden/infsup.npz)
must be reproduced regardless of the start vector."""
import os

import numpy as np
import pytest

from golden_io import GOLDEN

pytestmark = pytest.mark.gpu


def test_infsup_constants_vs_reference(gpu):
    from paper_2311_18461_b200.infsup import infsup_constant
    g = np.load(os.path.join(GOLDEN, "infsup.npz"))
    for (p, n), ls, gal in zip(g["cases"], g["ls"], g["galerkin"]):
        assert abs(infsup_constant("ls", int(p), int(n)) - ls) <= 1e-8 * ls
        assert abs(infsup_constant("galerkin", int(p), int(n)) - gal) <= 1e-8 * gal
