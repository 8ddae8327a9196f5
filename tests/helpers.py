"""Problem construction shared by the CPU and GPU tests: the host setup of
libks (ks_setup_*, pure host code) gives the bands and eigenpairs that both
the oracle and the GPU consume, so parity compares identical inputs."""
import numpy as np


def setup_arrays(ks, d, p, n_el, n_el_t, T=1.0, nu=1.0):
    prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el_t, T, nu)
    Lt, Mt, Wt = prob.time_bands()
    U, lam, M, L, G, V = [], [], [], [], [], []
    for l in range(d):
        u, lm = prob.eig(l)
        U.append(u)
        lam.append(lm)
        m, ll, g, v = prob.space_bands(l)
        M.append(m); L.append(ll); G.append(g); V.append(v)
    return dict(prob=prob, dims=prob.reduced_dims(), d=d, p=p, nu=nu, Lt=Lt, Mt=Mt, Wt=Wt,
                U=U, lam=lam, M=M, L=L, G=G, V=V)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def maxrel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
