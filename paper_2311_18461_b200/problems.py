"""Manufactured solutions of the BASELINE workloads as vectorised numpy
callables fn(t, x_1, ..., x_d) for Quadrature (restating the closed forms of
the reference's problems.cpp and the c2/c4 solution of SURVEY 8(d), G2):

    sinsin             u = prod_l sin(pi x_l) exp(-i d pi^2 t),  f = i u_t - nu lap u = (1 + nu) d pi^2 u
                       (4 pi^2 u at d = 2, nu = 1: SURVEY 8(d) c2/c4)
    traveling_wave_2d  u = a exp(-i (|x|^2 + t^2) / w^2), w = 0.2, a = (2 / w^2)^(1/4)  (problems.cpp:95-117)
"""
import numpy as np

PI = 3.14159265358979323846


def sinsin(d, nu=1.0):
    def u(t, *x):
        v = np.exp(-1j * d * PI * PI * t)
        for xi in x:
            v = v * np.sin(PI * xi)
        return v

    def f(t, *x):
        return (1.0 + nu) * d * PI * PI * u(t, *x)
    return u, f


def traveling_wave_2d():
    w = 0.2
    a = (2.0 / (w * w)) ** 0.25
    iw2 = 1.0 / (w * w)

    def u(t, x1, x2):
        r2 = x1 * x1 + x2 * x2
        return a * np.exp(-1j * (r2 + t * t) * iw2)

    def f(t, x1, x2):
        r2 = x1 * x1 + x2 * x2
        return u(t, x1, x2) * ((4.0 * r2 * iw2 * iw2 + 2.0 * t * iw2) + 4.0j * iw2)
    return u, f


def by_name(name, d):
    if name == "sinsin":
        return sinsin(d)
    if name == "traveling_wave_2d":
        return traveling_wave_2d()
    raise ValueError("unknown problem: " + name)
