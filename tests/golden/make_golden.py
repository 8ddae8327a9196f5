"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself:
/root/reference/proj/src/*.cpp compiled unmodified into oracle/_ref
(oracle/build_ref.sh), driven through oracle/ref_driver.cpp.

Run here (the reference tree exists only in the build container):
    bash oracle/build_ref.sh && python tests/golden/make_golden.py

Each case_*.npz holds the reference's setup products (reduced dims, time and
space bands, eigenpairs, composite eigenvalues), a seeded input r
(std::mt19937_64(1234), re/im = 2u-1), and the reference's outputs:
FD apply z = P^-1 r, matvec y = A r, one factored block (ab, piv), and a
PCG solve (iterations, residual history, x). Outputs are produced twice:
with the reference's scalar backend (bit-exact target for the C oracle) and
with its default AVX2 backend ("_avx2" keys, the reference as shipped).
tw_*.npz hold the 2-D traveling-wave right-hand sides of the paper's Table 2
(lift_nonhomogeneous) and the reference's FD-PCG counts.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import refdrv  # noqa: E402

CASES = [  # (d, p, n_el, n_el_t) -- reference unit-test shapes + config 1 + 3-D
    (1, 2, 5, 4), (2, 2, 3, 4), (1, 2, 1, 1), (1, 3, 6, 6), (1, 3, 64, 64),
    (2, 3, 10, 9), (2, 4, 6, 5), (2, 6, 5, 5), (3, 2, 6, 6), (3, 4, 4, 4),
]
TW = [(2, 8), (3, 8), (4, 8), (2, 16), (3, 16), (4, 16)]  # Table 2: 7 / 9 / 10 +- 2
# final-condition trial space (time basis drops its LAST function, assembly.hpp:59-62;
# SURVEY 8(f) rank 2): same Kronecker skeleton, different time restriction
FC_CASES = [(1, 2, 5, 4), (2, 3, 8, 7), (3, 2, 6, 6)]
# Galerkin fast solver (fdsolver.cpp:177-191) and Galerkin operator (assembly.cpp:273-286)
GAL_CASES = [(1, 2, 5, 4), (2, 3, 6, 5), (3, 2, 6, 6)]
# right-hand side, lifting, solution and error norms of manufactured solutions
# (assembly.cpp:390-404,514-570; experiments.cpp:73-153): (d, p, n_el, name)
RHS_CASES = [(1, 3, 8, "sinsin"), (2, 2, 6, "sinsin"), (2, 3, 6, "traveling_wave_2d"), (3, 2, 4, "sinsin")]


def case(d, p, n_el, n_el_t, trial=0):
    out = {"trial": trial}
    R = refdrv.RefProblem(d, p, n_el, n_el_t, trial=trial)
    Lt, Mt, Wt = R.time_bands()
    out.update(dims=np.array(R.dims), d=d, p=p, nu=1.0, Lt=Lt, Mt=Mt, Wt=Wt,
               lam_composite=R.composite_lambda())
    for l in range(d):
        U, lam = R.eig(l)
        M, L, G, V = R.space_bands(l)
        out.update({f"U{l}": U, f"lam{l}": lam, f"M{l}": M, f"L{l}": L, f"G{l}": G, f"V{l}": V})
    r = O.random_vec(R.N, 1234)
    out["r"] = r
    ns = R.N // R.dims[0]
    ab, piv = R.fd_block(ns // 2)
    out.update(block_index=ns // 2, block_ab=ab, block_piv=piv)
    for tag, be in (("", "scalar"), ("_avx2", "auto")):
        refdrv.force_backend(be)
        out["z" + tag] = R.fd_apply(r)
        out["y" + tag] = R.kron_apply(r)
        s = R.pcg(r, 1e-8, 200)
        out["pcg_iters" + tag] = s["iterations"]
        out["pcg_hist" + tag] = np.array(s["res_history"])
        out["pcg_x" + tag] = s["x"]
    refdrv.force_backend("scalar")
    return out


def galerkin_case(d, p, n_el, n_el_t):
    R = refdrv.RefProblem(d, p, n_el, n_el_t)
    Lt, Mt, Wt = R.time_bands()
    out = {"dims": np.array(R.dims), "p": p, "Lt": Lt, "Mt": Mt, "Wt": Wt}
    for l in range(d):
        U, lam = R.eig(l)
        M, L, G, V = R.space_bands(l)
        out.update({f"U{l}": U, f"lam{l}": lam, f"M{l}": M, f"L{l}": L, f"G{l}": G, f"V{l}": V})
    r = O.random_vec(R.N, 1234)
    refdrv.force_backend("scalar")
    out.update(r=r, z_gal=R.galerkin_apply(r), z_gal_adj=R.galerkin_apply(r, True), y_gal=R.galerkin_kron_apply(r))
    return out


def rhs_case(d, p, n_el, name):
    R = refdrv.RefProblem(d, p, n_el, n_el)
    refdrv.force_backend("scalar")
    b0 = R.assemble_rhs_named(name)
    rhs, bnd = R.lift_named(name)
    sol = R.pcg(rhs, 1e-10, 400)
    full = R.extend(sol["x"], bnd)
    l2, en = R.error_norms_named(name, full)
    return {"d": d, "p": p, "n_el": n_el, "name": name, "dims": np.array(R.dims), "rhs_f": b0, "rhs": rhs,
            "boundary": bnd, "x": sol["x"], "full": full, "l2": l2, "energy": en}


def main():
    for c in CASES:
        name = "case_d%d_p%d_n%d_t%d.npz" % c
        np.savez_compressed(os.path.join(HERE, name), **case(*c))
        print("wrote", name)
    for c in GAL_CASES:
        name = "gal_d%d_p%d_n%d_t%d.npz" % c
        np.savez_compressed(os.path.join(HERE, name), **galerkin_case(*c))
        print("wrote", name)
    for c in RHS_CASES:
        name = "rhs_d%d_p%d_n%d_%s.npz" % c
        np.savez_compressed(os.path.join(HERE, name), **rhs_case(*c))
        print("wrote", name)
    # inf-sup constants (experiments.cpp:185-232) on spaces small enough that
    # 60 Lanczos steps exhaust the Krylov space
    inf = {"cases": np.array([(p, n) for p in (2, 3) for n in (4, 6)]), "ls": [], "galerkin": []}
    for p, n in inf["cases"]:
        inf["ls"].append(refdrv.infsup("ls", int(p), int(n)))
        inf["galerkin"].append(refdrv.infsup("galerkin", int(p), int(n)))
    np.savez_compressed(os.path.join(HERE, "infsup.npz"), **inf)
    print("wrote infsup.npz")
    for c in FC_CASES:
        name = "case_fc_d%d_p%d_n%d_t%d.npz" % c
        np.savez_compressed(os.path.join(HERE, name), **case(*c, trial=1))
        print("wrote", name)
    for p, n_el in TW:
        R = refdrv.RefProblem(2, p, n_el, n_el)
        refdrv.force_backend("auto")
        b = R.named_rhs("traveling_wave_2d")
        s = R.pcg(b, 1e-8, 200)
        Lt, Mt, Wt = R.time_bands()
        d = {"dims": np.array(R.dims), "p": p, "b": b, "pcg_iters": s["iterations"],
             "Lt": Lt, "Mt": Mt, "Wt": Wt}
        for l in range(2):
            U, lam = R.eig(l)
            M, L, G, V = R.space_bands(l)
            d.update({f"U{l}": U, f"lam{l}": lam, f"M{l}": M, f"L{l}": L, f"G{l}": G, f"V{l}": V})
        name = "tw_p%d_n%d.npz" % (p, n_el)
        np.savez_compressed(os.path.join(HERE, name), **d)
        print("wrote", name, "iters", s["iterations"])
    refdrv.force_backend("scalar")


if __name__ == "__main__":
    main()
