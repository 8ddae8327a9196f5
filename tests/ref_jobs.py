"""Reference-side jobs for the full-size parity tests (tests/test_gpu_full_configs.py).

Each job builds the problem with the reference's OWN code (oracle/_ref: the
unmodified reference sources, oracle/build_ref.sh) and returns its outputs on
seeded inputs. The jobs run in separate worker processes (the reference is
single-threaded) so the GPU tests can wait on them concurrently. Test
infrastructure only: nothing here is imported by the product package.

Reference entry points: FDPreconditioner::apply (fdsolver.cpp:53-63),
KroneckerOperator::apply (tensorops.cpp:236-254), pcg (krylov.cpp:24-114),
lift_nonhomogeneous (assembly.cpp:514-570), error_norms (experiments.cpp:73-153).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ref(d, p, n_el, n_el_t, with_fd=True):
    from oracle import refdrv
    if not refdrv.available():
        raise RuntimeError("oracle/_ref/libkronschro_ref.so missing (run __graft_entry__.build())")
    return refdrv.RefProblem(d, p, n_el, n_el_t, with_fd=with_fd)


def apply_job(d, p, n_el, n_el_t, seed):
    """One FD application and one system matvec on the seeded random vector."""
    from oracle import oracle as O
    ref = _ref(d, p, n_el, n_el_t)
    r = O.random_vec(ref.N, seed)
    return {"dims": ref.dims, "z": ref.fd_apply(r), "y": ref.kron_apply(r)}


def random_solve_job(d, p, n_el, n_el_t, seed, tol=1e-8, maxit=200):
    """FD-preconditioned CG on the seeded random right-hand side."""
    from oracle import oracle as O
    ref = _ref(d, p, n_el, n_el_t)
    b = O.random_vec(ref.N, seed)
    rep = ref.pcg(b, tol=tol, maxit=maxit)
    return {"dims": ref.dims, "iterations": rep["iterations"], "converged": rep["converged"],
            "breakdown": rep["breakdown"], "res_history": rep["res_history"], "x": rep["x"]}


def manufactured_job(d, p, n_el, n_el_t, keep_x=True):
    """BASELINE configs[1] / [3]: sin-sin manufactured solution, lifted right-hand
    side, FD-PCG to 1e-8, extension with the boundary values, L2 / energy errors."""
    ref = _ref(d, p, n_el, n_el_t)
    rhs, bnd = ref.lift_named("sinsin")
    rep = ref.pcg(rhs, tol=1e-8, maxit=200)
    full = ref.extend(rep["x"], bnd)
    l2, en = ref.error_norms_named("sinsin", full)
    out = {"dims": ref.dims, "iterations": rep["iterations"], "converged": rep["converged"],
           "l2": l2, "energy": en, "res_history": rep["res_history"]}
    if keep_x:
        out.update(rhs=rhs, bnd=bnd, x=rep["x"], full=full)
    return out


def restart_job(d, p, n_el, n_el_t, seed, tol):
    """A tolerance below the attainable accuracy: the recurrence residual drops
    under tol while the true residual does not, so pcg restarts from the exact
    residual (krylov.cpp:84-100) and gives up after the third time."""
    from oracle import oracle as O
    ref = _ref(d, p, n_el, n_el_t)
    b = O.random_vec(ref.N, seed)
    rep = ref.pcg(b, tol=tol, maxit=400)
    return {"iterations": rep["iterations"], "converged": rep["converged"],
            "breakdown": rep["breakdown"], "res_history": rep["res_history"]}
