"""kronschro-b200: B200 (sm_100a) hot path of the space-time least-squares
isogeometric Schroedinger solver (arXiv 2311.18461), behind the C-ABI in
include/ks.h (libks.so, built in-tree by ``make -C paper_2311_18461_b200``).

Python mirror of the reference's solver API for this path (reference
proj/include/kronschro/*.hpp), with the same names, argument meaning and
error behaviour:

    SpaceTimeProblem.uniform(d, p, n_el, n_el_time, T, nu)   assembly.hpp:29-63
    FDPreconditioner(prob)          .apply(r) -> z           fdsolver.hpp:56-74
    KroneckerOperator(dims)         .add_term / .apply       tensorops.hpp:57-87
    assemble_system_operator(prob)                           assembly.hpp:76
    pcg(A, P, b, PcgOptions) -> SolveReport                  krylov.hpp:11-38

All arithmetic runs in libks.so on the GPU. There is no CPU fallback: without
the extension or without a CUDA device, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KS_LIB_PATH") or os.path.join(_HERE, "libks.so")  # override: experiment builds

KS_OK, KS_EINVAL, KS_ESINGULAR, KS_ECUDA, KS_ENOMEM, KS_ENCCL, KS_ELENGTH = range(7)
KS_MEM_HOST, KS_MEM_DEVICE = 0, 1


class KsError(RuntimeError):
    code = -1


class InvalidArgument(KsError, ValueError):
    """std::invalid_argument in the reference."""
    code = KS_EINVAL


class SingularError(KsError):
    """std::runtime_error('factor_banded: numerically singular pivot')."""
    code = KS_ESINGULAR


class CudaError(KsError):
    code = KS_ECUDA


class DeviceMemoryError(KsError, MemoryError):
    code = KS_ENOMEM


class LengthError(KsError, ValueError):
    """std::length_error (dense caps)."""
    code = KS_ELENGTH


_ERR = {KS_EINVAL: InvalidArgument, KS_ESINGULAR: SingularError, KS_ECUDA: CudaError,
        KS_ENOMEM: DeviceMemoryError, KS_ELENGTH: LengthError}


class ks_c64(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


class ks_term(C.Structure):
    _fields_ = [("coeff", ks_c64), ("factors", C.POINTER(C.c_void_p)),
                ("bw", C.POINTER(C.c_int))]


class ks_pcg_opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("maxit", C.c_int), ("strict_residual", C.c_int)]


class ks_pcg_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("restarts", C.c_int), ("hist_len", C.c_int),
                ("matvec_seconds", C.c_double), ("precond_seconds", C.c_double),
                ("solve_seconds", C.c_double)]


# every symbol include/ks.h declares, with its ctypes signature
_P = C.c_void_p
_SIGS = {
    "ks_last_error": (C.c_char_p, []),
    "ks_version": (C.c_int, []),
    "ks_device_count": (C.c_int, []),
    "ks_fd_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_double, C.c_int, C.POINTER(_P),
                               C.POINTER(_P), _P, _P, _P, C.c_int, C.POINTER(_P)]),
    "ks_fd_apply": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "ks_fd_apply_adjoint": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "ks_fd_vec_size": (C.c_size_t, [_P]),
    "ks_fd_eigenvalues": (C.c_int, [_P, _P]),
    "ks_fd_block": (C.c_int, [_P, C.c_size_t, _P, _P]),
    "ks_fd_info": (C.c_int, [_P, _P, _P]),
    "ks_fd_destroy": (C.c_int, [_P]),
    "ks_kron_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(ks_term),
                                 C.c_int, C.POINTER(_P)]),
    "ks_kron_apply": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "ks_kron_vec_size": (C.c_size_t, [_P]),
    "ks_kron_plan_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int)]),
    "ks_kron_engine": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "ks_kron_destroy": (C.c_int, [_P]),
    "ks_pcg_sharded": (C.c_int, [_P, _P, _P, _P, _P, C.c_int, C.POINTER(ks_pcg_opts), _P, C.c_int,
                                 C.POINTER(ks_pcg_report)]),
    "ks_pcg": (C.c_int, [_P, _P, _P, _P, C.c_int, C.POINTER(ks_pcg_opts), _P, C.c_int,
                         C.POINTER(ks_pcg_report)]),
    "ks_axpy_real": (C.c_int, [C.c_double, _P, _P, C.c_size_t, _P]),
    "ks_axpy": (C.c_int, [ks_c64, _P, _P, C.c_size_t, _P]),
    "ks_dotc": (C.c_int, [_P, _P, C.c_size_t, C.POINTER(ks_c64), _P]),
    "ks_norm2sq": (C.c_int, [_P, C.c_size_t, C.POINTER(C.c_double), _P]),
    "ks_set_device": (C.c_int, [C.c_int]),
    "ks_malloc": (C.c_int, [C.POINTER(_P), C.c_size_t]),
    "ks_free": (C.c_int, [_P]),
    "ks_memcpy": (C.c_int, [_P, _P, C.c_size_t, C.c_int]),
    "ks_host_alloc": (C.c_int, [C.POINTER(_P), C.c_size_t]),
    "ks_host_free": (C.c_int, [_P]),
    "ks_synchronize": (C.c_int, []),
    "ks_stream_create": (C.c_int, [C.POINTER(_P)]),
    "ks_stream_destroy": (C.c_int, [_P]),
    "ks_stream_synchronize": (C.c_int, [_P]),
    "ks_flush_l2": (C.c_int, [C.c_size_t]),
    "ks_fd_time": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.POINTER(C.c_double),
                             C.POINTER(C.c_double)]),
    "ks_kron_time": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "ks_fd_latency": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "ks_fd_profile": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_int)]),
    "ks_fp64_peak": (C.c_int, [C.POINTER(C.c_double)]),
    "ks_fp64_peaks": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "ks_fp64_peak_mixed": (C.c_int, [C.POINTER(C.c_double)]),
    "ks_fp64_peak_mma16": (C.c_int, [C.POINTER(C.c_double)]),
    "ks_fp64_dmma_occupancy": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double)]),
    "ks_bw_fan": (C.c_int, [C.c_int, C.c_int, C.c_size_t, C.POINTER(C.c_double)]),
    "ks_transform_engine": (C.c_int, []),
    "ks_launch_count": (C.c_uint64, []),
    "ks_launch_count_reset": (None, []),
    "ks_shard_plan": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int,
                                C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "ks_fdshard_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_double, C.c_int,
                                    C.POINTER(_P), C.POINTER(_P), _P, _P, _P, C.c_int, C.c_int,
                                    C.c_int, C.POINTER(_P)]),
    "ks_fdshard_sizes": (C.c_int, [_P, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "ks_fdshard_forward": (C.c_int, [_P, _P, _P, _P]),
    "ks_fdshard_middle": (C.c_int, [_P, _P, _P]),
    "ks_fdshard_backward": (C.c_int, [_P, _P, _P, _P]),
    "ks_fdshard_forward_slab": (C.c_int, [_P, _P, _P, _P]),
    "ks_fdshard_set_peers": (C.c_int, [_P, _P, _P]),
    "ks_fdshard_middle_peer": (C.c_int, [_P, _P]),
    "ks_fdshard_backward_slab": (C.c_int, [_P, _P, _P, _P]),
    "ks_ipc_get_handle": (C.c_int, [_P, _P]),
    "ks_ipc_open": (C.c_int, [_P, C.POINTER(_P)]),
    "ks_ipc_close": (C.c_int, [_P]),
    "ks_fdshard_destroy": (C.c_int, [_P]),
    "ks_comm_unique_id": (C.c_int, [_P]),
    "ks_comm_create": (C.c_int, [C.c_int, C.c_int, _P, C.c_int, C.POINTER(C.c_void_p)]),
    "ks_comm_destroy": (C.c_int, [_P]),
    "ks_fdshard_apply": (C.c_int, [_P, _P, _P, _P, _P]),
    "ks_kronshard_apply_comm": (C.c_int, [_P, _P, _P, _P, _P]),
    "ks_kronshard_create": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(ks_term),
                                      C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "ks_kronshard_sizes": (C.c_int, [_P, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                     C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                     C.POINTER(C.c_size_t)]),
    "ks_kronshard_apply": (C.c_int, [_P, _P, _P, _P]),
    "ks_kronshard_plan": (C.c_int, [C.c_longlong, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_longlong),
                                    C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                    C.POINTER(C.c_longlong)]),
    "ks_cg_update": (C.c_int, [C.c_double, _P, _P, _P, _P, C.c_size_t, C.POINTER(C.c_double), _P]),
    "ks_xpby": (C.c_int, [_P, C.c_double, _P, C.c_size_t, _P]),
    "ks_setup_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                  C.c_int, C.POINTER(_P)]),
    "ks_setup_dims": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ks_setup_time_bands": (C.c_int, [_P, _P, _P, _P]),
    "ks_setup_space_bands": (C.c_int, [_P, C.c_int, _P, _P, _P, _P]),
    "ks_setup_eig": (C.c_int, [_P, C.c_int, _P, _P]),
    "ks_setup_create_fd": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "ks_setup_create_system": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "ks_setup_create_galerkin_fd": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "ks_setup_full_dims": (C.c_int, [_P, _P]),
    "ks_setup_quad_rule": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), _P, _P]),
    "ks_setup_greville": (C.c_int, [_P, C.c_int, C.POINTER(C.c_int), _P]),
    "ks_quad_create": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "ks_quad_destroy": (C.c_int, [_P]),
    "ks_quad_dims": (C.c_int, [_P, _P, C.POINTER(C.c_int), _P]),
    "ks_quad_rhs_reset": (C.c_int, [_P]),
    "ks_quad_rhs_named": (C.c_int, [_P, C.c_char_p, _P, C.c_int]),
    "ks_quad_sample_named": (C.c_int, [_P, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    "ks_quad_rhs_chunk": (C.c_int, [_P, C.c_int, C.c_int, _P, C.c_int]),
    "ks_quad_rhs_finish": (C.c_int, [_P, _P, C.c_int]),
    "ks_quad_lift": (C.c_int, [_P, _P, C.c_int, _P, _P]),
    "ks_quad_extend": (C.c_int, [_P, _P, _P, C.c_int, _P]),
    "ks_quad_initial_term": (C.c_int, [_P, _P, C.c_int, _P, C.c_int]),
    "ks_quad_error_set": (C.c_int, [_P, _P, C.c_int]),
    "ks_quad_error_chunk": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, C.c_int, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]),
    "ks_setup_create_galerkin_operator": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "ks_fd_create_galerkin": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_double, C.c_int, C.POINTER(_P),
                                        C.POINTER(_P), _P, _P, C.c_int, C.POINTER(_P)]),
    "ks_setup_create_system_sharded": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "ks_setup_destroy": (C.c_int, [_P]),
}

_lib = None


def lib():
    """Load libks.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libks.so not built: run `make -C {_HERE}` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int):
    if rc != KS_OK:
        msg = lib().ks_last_error().decode(errors="replace")
        raise _ERR.get(rc, KsError)(msg)


def device_count() -> int:
    return lib().ks_device_count()


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _cvec(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _stream(stream):
    """A ks.Stream, a raw cudaStream_t (int / c_void_p) or None -> ctypes argument."""
    return stream.handle if isinstance(stream, Stream) else stream


def _dev_pair(n, x, y, what):
    """Check device vectors against the operator size; allocate y if absent."""
    if x.n != n:
        raise InvalidArgument(f"{what}: vector length mismatch ({x.n} != {n})")
    if y is None:
        return DeviceVector(n)
    if not isinstance(y, DeviceVector) or y.n != n:
        raise InvalidArgument(f"{what}: output must be a DeviceVector of length {n}")
    return y


def _host_out(n, y, what):
    """Output array for a host-pointer apply: a new one, or the caller's if it is
    a C-contiguous complex128 array of length n (the D2H copy writes n entries)."""
    if y is None:
        return np.empty(n, dtype=np.complex128)
    if not (isinstance(y, np.ndarray) and y.dtype == np.complex128 and y.flags["C_CONTIGUOUS"] and y.size == n
            and y.flags["WRITEABLE"]):
        raise InvalidArgument(f"{what}: output must be a writeable C-contiguous complex128 array of length {n}")
    return y


# ---------------------------------------------------------------------------
# device buffers (HBM-resident vectors for the device-pointer API)
# ---------------------------------------------------------------------------
class DeviceVector:
    """A complex128 vector in device memory (libks allocation)."""

    def __init__(self, n: int):
        self.n = int(n)
        self.nbytes = self.n * 16
        p = C.c_void_p()
        _check(lib().ks_malloc(C.byref(p), max(self.nbytes, 16)))
        self.ptr = p

    @classmethod
    def from_host(cls, a: np.ndarray) -> "DeviceVector":
        a = _cvec(a).ravel()
        v = cls(a.size)
        _check(lib().ks_memcpy(v.ptr, _ptr(a), v.nbytes, 0))
        return v

    def to_host(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.complex128)
        _check(lib().ks_memcpy(_ptr(out), self.ptr, self.nbytes, 1))
        return out

    def copy_from(self, a: np.ndarray):
        a = _cvec(a).ravel()
        assert a.size == self.n
        _check(lib().ks_memcpy(self.ptr, _ptr(a), self.nbytes, 0))

    def __del__(self):
        try:
            if getattr(self, "ptr", None) is not None and self.ptr.value:
                lib().ks_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# SpaceTimeProblem + UnivariateSet mirror (host setup in libks, assembly.cpp)
# ---------------------------------------------------------------------------
class SpaceTimeProblem:
    """Uniform space-time problem: SpaceTimeProblem::uniform (assembly.cpp:110-117)."""

    def __init__(self, handle, d, p, dims, T, nu, trial):
        self._h = handle
        self.d, self.p, self.T, self.nu, self.trial = d, p, T, nu, trial
        self.dims = list(dims)

    @classmethod
    def uniform(cls, d: int, p: int, n_el: int, n_el_time: int, T: float = 1.0,
                nu: float = 1.0, trial: str = "initial") -> "SpaceTimeProblem":
        h = C.c_void_p()
        tr = {"initial": 0, "final": 1}[trial]
        _check(lib().ks_setup_create(d, p, n_el, n_el_time, T, nu, tr, C.byref(h)))
        dd, pp = C.c_int(), C.c_int()
        dims = (C.c_int * (d + 1))()
        _check(lib().ks_setup_dims(h, C.byref(dd), dims, C.byref(pp)))
        return cls(h, d, p, list(dims), T, nu, trial)

    @classmethod
    def matched(cls, d, p, n_el, T=1.0, nu=1.0, trial="initial"):
        """SpaceTimeProblem::matched (assembly.cpp:119-123)."""
        return cls.uniform(d, p, n_el, max(1, int(round(n_el * T))), T, nu, trial)

    def reduced_dims(self) -> List[int]:
        return list(self.dims)

    @property
    def n_t(self) -> int:
        return self.dims[0]

    def n_s(self, l: int) -> int:
        return self.dims[l + 1]

    @property
    def N_s(self) -> int:
        return int(np.prod(self.dims[1:]))

    @property
    def N_dof(self) -> int:
        return self.N_s * self.n_t

    def time_bands(self):
        nt, p = self.dims[0], self.p
        Lt = np.zeros((nt, 2 * p + 1))
        Mt = np.zeros((nt, 2 * p + 1))
        Wt = np.zeros((nt, 2 * p + 1), dtype=np.complex128)
        _check(lib().ks_setup_time_bands(self._h, _ptr(Lt), _ptr(Mt), _ptr(Wt)))
        return Lt.ravel(), Mt.ravel(), Wt.ravel()

    def space_bands(self, l: int):
        n, p = self.dims[l + 1], self.p
        out = [np.zeros((n, 2 * p + 1)) for _ in range(4)]
        _check(lib().ks_setup_space_bands(self._h, l, *[_ptr(a) for a in out]))
        return tuple(a.ravel() for a in out)  # M, L, G, V

    def eig(self, l: int):
        n = self.dims[l + 1]
        U = np.zeros(n * n)
        lam = np.zeros(n)
        _check(lib().ks_setup_eig(self._h, l, _ptr(U), _ptr(lam)))
        return U, lam

    def __del__(self):
        try:
            if self._h:
                lib().ks_setup_destroy(self._h)
                self._h = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# FD preconditioner
# ---------------------------------------------------------------------------
class Stream:
    """A CUDA stream for asynchronous applies (host-pointer applies on a stream
    are pipelined; results are valid after synchronize())."""

    def __init__(self):
        h = C.c_void_p()
        _check(lib().ks_stream_create(C.byref(h)))
        self.handle = h

    def synchronize(self):
        _check(lib().ks_stream_synchronize(self.handle))

    def __del__(self):
        try:
            if self.handle:
                lib().ks_stream_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class FDPreconditioner:
    """Fast-diagonalisation preconditioner (fdsolver.hpp:56-74) on the GPU.

    FDPreconditioner(prob) uses the host setup of ``prob``;
    FDPreconditioner.from_arrays(...) takes the reference's own setup products
    (U_l, lambda_l, Lt, Mt, Wt), which is how a reference process drops it in.
    """

    def __init__(self, prob: Optional[SpaceTimeProblem] = None, device: int = 0, _handle=None,
                 _dims=None):
        if _handle is not None:
            self._h = _handle
            self.dims = list(_dims)
        else:
            h = C.c_void_p()
            _check(lib().ks_setup_create_fd(prob._h, device, C.byref(h)))
            self._h = h
            self.dims = prob.reduced_dims()
        self.device = device

    @classmethod
    def galerkin(cls, prob: "SpaceTimeProblem", device: int = 0) -> "FDPreconditioner":
        """galerkin_fast_solver(prob, u) (fdsolver.hpp:76-79, fdsolver.cpp:177-191): exact
        inverse of the Galerkin matrix; apply = solve, apply_adjoint = solve_adjoint."""
        h = C.c_void_p()
        _check(lib().ks_setup_create_galerkin_fd(prob._h, device, C.byref(h)))
        return cls(device=device, _handle=h, _dims=prob.reduced_dims())

    @classmethod
    def galerkin_from_arrays(cls, dims: Sequence[int], nu: float, p_t: int, U: Sequence[np.ndarray],
                             lam: Sequence[np.ndarray], Mt, Wt, device: int = 0):
        d = len(dims) - 1
        Us = [np.ascontiguousarray(u, dtype=np.float64).ravel() for u in U]
        ls = [np.ascontiguousarray(v, dtype=np.float64).ravel() for v in lam]
        Mt = np.ascontiguousarray(Mt, dtype=np.float64).ravel()
        Wt = _cvec(Wt).ravel()
        up = (C.c_void_p * d)(*[a.ctypes.data for a in Us])
        lp = (C.c_void_p * d)(*[a.ctypes.data for a in ls])
        cd = (C.c_int * (d + 1))(*dims)
        h = C.c_void_p()
        _check(lib().ks_fd_create_galerkin(d, cd, float(nu), int(p_t), up, lp, _ptr(Mt), _ptr(Wt), device,
                                           C.byref(h)))
        return cls(device=device, _handle=h, _dims=dims)

    @classmethod
    def from_arrays(cls, dims: Sequence[int], nu: float, p_t: int, U: Sequence[np.ndarray],
                    lam: Sequence[np.ndarray], Lt, Mt, Wt, device: int = 0):
        d = len(dims) - 1
        Us = [np.ascontiguousarray(u, dtype=np.float64).ravel() for u in U]
        ls = [np.ascontiguousarray(v, dtype=np.float64).ravel() for v in lam]
        Lt = np.ascontiguousarray(Lt, dtype=np.float64).ravel()
        Mt = np.ascontiguousarray(Mt, dtype=np.float64).ravel()
        Wt = _cvec(Wt).ravel()
        up = (C.c_void_p * d)(*[a.ctypes.data for a in Us])
        lp = (C.c_void_p * d)(*[a.ctypes.data for a in ls])
        cd = (C.c_int * (d + 1))(*dims)
        h = C.c_void_p()
        _check(lib().ks_fd_create(d, cd, float(nu), int(p_t), up, lp, _ptr(Lt), _ptr(Mt), _ptr(Wt),
                                  device, C.byref(h)))
        return cls(device=device, _handle=h, _dims=dims)

    def vec_size(self) -> int:
        return int(lib().ks_fd_vec_size(self._h))

    def apply(self, r, z=None, stream=None):
        """z = P^-1 r. numpy in -> numpy out (host path), or DeviceVector in/out."""
        n = self.vec_size()
        if isinstance(r, DeviceVector):
            z = _dev_pair(n, r, z, "FastDiagSolver")
            _check(lib().ks_fd_apply(self._h, r.ptr, z.ptr, KS_MEM_DEVICE, _stream(stream)))
            return z
        r = _cvec(r).ravel()
        if r.size != n:
            raise InvalidArgument("FastDiagSolver: vector length mismatch")
        out = _host_out(n, z, "FastDiagSolver")
        _check(lib().ks_fd_apply(self._h, _ptr(r), _ptr(out), KS_MEM_HOST, _stream(stream)))
        return out

    def apply_adjoint(self, r):
        r = _cvec(r).ravel()
        if r.size != self.vec_size():
            raise InvalidArgument("FastDiagSolver: vector length mismatch")
        out = np.empty_like(r)
        _check(lib().ks_fd_apply_adjoint(self._h, _ptr(r), _ptr(out), KS_MEM_HOST, None))
        return out

    def eigenvalues(self) -> np.ndarray:
        out = np.zeros(int(np.prod(self.dims[1:])))
        _check(lib().ks_fd_eigenvalues(self._h, _ptr(out)))
        return out

    def block(self, i: int, p: int):
        nt = self.dims[0]
        ab = np.zeros(nt * (3 * p + 1), dtype=np.complex128)
        piv = np.zeros(nt, dtype=np.int32)
        _check(lib().ks_fd_block(self._h, int(i), _ptr(ab), _ptr(piv)))
        return ab, piv

    def info(self) -> dict:
        """Execution plan: axes on the folded (even/odd) transform, factored blocks."""
        m, nb = C.c_int(), C.c_size_t()
        _check(lib().ks_fd_info(self._h, C.byref(m), C.byref(nb)))
        d = len(self.dims) - 1
        return {"folded_axes": [l + 1 for l in range(d) if m.value >> l & 1], "blocks": nb.value,
                "time_major_axis": 1 if m.value >> 17 & 1 else d,
                # least-squares blocks: L D L^H (never pivots); Galerkin LU: no block pivoted
                "no_pivot_solve": bool(m.value >> 18 & 1),
                # axis-1 transform + block solves + inverse transform in one kernel (ks_fdaxis1.cu)
                "fused_axis1": bool(m.value >> 19 & 1)}

    def latency(self, r: DeviceVector, z: DeviceVector, iters: int = 100, graph: bool = True) -> float:
        """ms per apply over `iters` back-to-back applies (CUDA-graph replays if graph)."""
        ms = C.c_double()
        _check(lib().ks_fd_latency(self._h, r.ptr, z.ptr, int(iters), int(graph), C.byref(ms)))
        return ms.value

    def profile(self, r: DeviceVector, z: DeviceVector, iters: int, flush: bool = False) -> dict:
        """ms per apply, and the device time per apply split by kernel kind
        (CUDA events around every launch) with the launch counts."""
        ms = C.c_double()
        mk = (C.c_double * 3)()
        nl = (C.c_int * 3)()
        _check(lib().ks_fd_profile(self._h, r.ptr, z.ptr, iters, int(flush), C.byref(ms), mk, nl))
        names = ("transforms", "fused_axis1", "solves")
        return {"ms": ms.value, **{n: {"ms": mk[i], "launches": nl[i]} for i, n in enumerate(names)}}

    def time(self, r: DeviceVector, z: DeviceVector, iters: int, flush: bool = True):
        ms, mk = C.c_double(), C.c_double()
        _check(lib().ks_fd_time(self._h, r.ptr, z.ptr, iters, int(flush), C.byref(ms),
                                C.byref(mk)))
        return ms.value, mk.value

    def __del__(self):
        try:
            if self._h:
                lib().ks_fd_destroy(self._h)
                self._h = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Kronecker operator
# ---------------------------------------------------------------------------
class Banded:
    """BandedMatrix<cplx> (banded.hpp): data[bw + i - j + j*(2bw+1)]."""

    def __init__(self, n: int, bw: int, data=None):
        if n < 1 or bw < 0:
            raise InvalidArgument("BandedMatrix: invalid dimensions")
        self.n, self.bw = n, bw
        self.data = (_cvec(data).ravel().copy() if data is not None
                     else np.zeros((2 * bw + 1) * n, dtype=np.complex128))
        if self.data.size != (2 * bw + 1) * n:
            raise InvalidArgument("BandedMatrix: data size mismatch")

    def to_dense(self) -> np.ndarray:
        n, bw = self.n, self.bw
        D = np.zeros((n, n), dtype=np.complex128)
        for j in range(n):
            for i in range(max(0, j - bw), min(n, j + bw + 1)):
                D[i, j] = self.data[bw + i - j + j * (2 * bw + 1)]
        return D

    @classmethod
    def from_dense(cls, D: np.ndarray, bw: int) -> "Banded":
        n = D.shape[0]
        b = cls(n, bw)
        for j in range(n):
            for i in range(max(0, j - bw), min(n, j + bw + 1)):
                b.data[bw + i - j + j * (2 * bw + 1)] = D[i, j]
        return b


class KroneckerOperator:
    """Sum of coeff * kron(F_D, ..., F_0) (tensorops.hpp:57-87) on the GPU."""

    def __init__(self, dims: Sequence[int], device: int = 0):
        for v in dims:
            if v < 1:
                raise InvalidArgument("CoeffTensor: dims must be positive")
        self._dims = list(dims)
        self.device = device
        self.terms = []  # (coeff, [Banded|None])
        self._h = None

    @classmethod
    def _wrap(cls, handle, dims, device):
        k = cls(dims, device)
        k._h = handle
        k.terms = None
        return k

    def dims(self):
        return list(self._dims)

    def vec_size(self) -> int:
        return int(np.prod(self._dims))

    def add_term(self, coeff: complex, factors: Sequence[Optional[Banded]]):
        """KroneckerOperator::add_term (tensorops.cpp:219-234)."""
        if self.terms is None:
            raise InvalidArgument("operator built from a fixed term list")
        if len(factors) != len(self._dims):
            raise InvalidArgument("KroneckerOperator: wrong factor count")
        for k, f in enumerate(factors):
            if f is not None and f.n != self._dims[k]:
                raise InvalidArgument("KroneckerOperator: factor size mismatch")
        self.terms.append((complex(coeff), list(factors)))
        self._release()

    def _release(self):
        if self._h:
            lib().ks_kron_destroy(self._h)
            self._h = None

    def _build(self):
        if self._h:
            return
        D = len(self._dims)
        keep = []
        terms = (ks_term * max(1, len(self.terms)))()
        for t, (c, fs) in enumerate(self.terms):
            ptrs = (C.c_void_p * D)(*[f.data.ctypes.data if f is not None else None for f in fs])
            bws = (C.c_int * D)(*[f.bw if f is not None else 0 for f in fs])
            keep += [ptrs, bws]
            terms[t].coeff = ks_c64(c.real, c.imag)
            terms[t].factors = C.cast(ptrs, C.POINTER(C.c_void_p))
            terms[t].bw = C.cast(bws, C.POINTER(C.c_int))
        h = C.c_void_p()
        cd = (C.c_int * D)(*self._dims)
        _check(lib().ks_kron_create(D, cd, len(self.terms), terms, self.device, C.byref(h)))
        self._h = h

    def apply(self, x, y=None, stream=None):
        """y = K x (tensorops.cpp:236-254)."""
        self._build()
        n = self.vec_size()
        if isinstance(x, DeviceVector):
            y = _dev_pair(n, x, y, "KroneckerOperator")
            _check(lib().ks_kron_apply(self._h, x.ptr, y.ptr, KS_MEM_DEVICE, _stream(stream)))
            return y
        x = _cvec(x).ravel()
        if x.size != n:
            raise InvalidArgument("KroneckerOperator: vector length mismatch")
        out = _host_out(n, y, "KroneckerOperator")
        _check(lib().ks_kron_apply(self._h, _ptr(x), _ptr(out), KS_MEM_HOST, _stream(stream)))
        return out

    def plan_info(self):
        self._build()
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        _check(lib().ks_kron_plan_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        e = C.c_int()
        _check(lib().ks_kron_engine(self._h, C.byref(e)))
        return {"passes": a.value, "nodes": b.value, "products": c.value,
                "engine": {0: "level_passes", 1: "fused_pairs"}[e.value]}

    def time(self, x: DeviceVector, y: DeviceVector, iters: int, flush: bool = True):
        self._build()
        ms = C.c_double()
        _check(lib().ks_kron_time(self._h, x.ptr, y.ptr, iters, int(flush), C.byref(ms)))
        return ms.value

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass


def assemble_system_operator(prob: SpaceTimeProblem, device: int = 0) -> KroneckerOperator:
    """A = M_s x L_t + nu^2 B_s x M_t + nu L_s x (W_t + W_t^*) (assembly.cpp:202-257)."""
    h = C.c_void_p()
    _check(lib().ks_setup_create_system(prob._h, device, C.byref(h)))
    return KroneckerOperator._wrap(h, prob.reduced_dims(), device)


def assemble_galerkin_operator(prob: SpaceTimeProblem, device: int = 0) -> KroneckerOperator:
    """Galerkin matrix M_s x W_t - nu sum_l (..G_l^T..) x M_t (assembly.cpp:273-286)."""
    h = C.c_void_p()
    _check(lib().ks_setup_create_galerkin_operator(prob._h, device, C.byref(h)))
    return KroneckerOperator._wrap(h, prob.reduced_dims(), device)


# ---------------------------------------------------------------------------
# Right-hand side, lifting, error norms
# ---------------------------------------------------------------------------
class Quadrature:
    """Device-side assemble_rhs / lift_nonhomogeneous / extend_with_boundary /
    error_norms (assembly.cpp:390-404,468-490,514-570; experiments.cpp:73-153)
    for a SpaceTimeProblem. Functions are vectorised numpy callables
    fn(t, x_1, ..., x_d) returning complex arrays (broadcast over the grid);
    they are sampled on the host, chunk by chunk along the outermost axis, and
    every contraction / solve / operator / reduction runs on the GPU."""

    def __init__(self, prob: "SpaceTimeProblem", device: int = 0):
        self.prob = prob
        self.d = prob.d
        h = C.c_void_p()
        _check(lib().ks_quad_create(prob._h, device, C.byref(h)))
        self._h = h
        D = self.d + 1
        nq = (C.c_int * D)()
        fd = (C.c_int * D)()
        ch = C.c_int()
        _check(lib().ks_quad_dims(h, nq, C.byref(ch), fd))
        self.nq, self.chunk, self.full_dims = list(nq), ch.value, list(fd)
        self.nodes, self.weights, self.greville = [], [], []
        for a in range(D):
            n = C.c_int()
            x = np.zeros(self.nq[a])
            w = np.zeros(self.nq[a])
            _check(lib().ks_setup_quad_rule(prob._h, a, C.byref(n), _ptr(x), _ptr(w)))
            self.nodes.append(x)
            self.weights.append(w)
            g = np.zeros(self.full_dims[a])
            _check(lib().ks_setup_greville(prob._h, a, C.byref(n), _ptr(g)))
            self.greville.append(g)
        self.N_full = int(np.prod(self.full_dims))

    @staticmethod
    def _sample(fn, coords):
        """fn on the tensor grid of coords (axis 0 = time fastest) -> flat complex array."""
        D = len(coords)
        args = []
        for a, c in enumerate(coords):
            shape = [1] * D
            shape[D - 1 - a] = len(c)
            args.append(np.asarray(c, dtype=np.float64).reshape(shape))
        v = np.asarray(fn(*args), dtype=np.complex128)
        v = np.broadcast_to(v, tuple(len(c) for c in reversed(coords)))
        return np.ascontiguousarray(v).ravel()

    def _chunks(self):
        last = self.nq[self.d]
        for r0 in range(0, last, self.chunk):
            yield r0, min(last, r0 + self.chunk)

    def _chunk_buf(self):
        if getattr(self, "_cbuf", None) is None:
            n = int(np.prod(self.nq[:self.d])) * self.chunk
            self._cbuf = DeviceVector(n)
            self._cbuf2 = DeviceVector(n)
        return self._cbuf, self._cbuf2

    def assemble_rhs(self, f) -> np.ndarray:
        """f: vectorised callable (host sampling), or the name of a built-in
        manufactured solution ("sinsin", "traveling_wave_2d": device sampling)."""
        if isinstance(f, str):
            out = np.zeros(self.prob.N_dof, dtype=np.complex128)
            _check(lib().ks_quad_rhs_named(self._h, f.encode(), _ptr(out), KS_MEM_HOST))
            return out
        _check(lib().ks_quad_rhs_reset(self._h))
        for r0, r1 in self._chunks():
            if isinstance(f, str):
                b, _ = self._chunk_buf()
                _check(lib().ks_quad_sample_named(self._h, f.encode(), 1, 0, r0, r1, b.ptr))
                _check(lib().ks_quad_rhs_chunk(self._h, r0, r1, b.ptr, KS_MEM_DEVICE))
            else:
                coords = self.nodes[:self.d] + [self.nodes[self.d][r0:r1]]
                fs = self._sample(f, coords)
                _check(lib().ks_quad_rhs_chunk(self._h, r0, r1, _ptr(fs), KS_MEM_HOST))
        out = np.zeros(self.prob.N_dof, dtype=np.complex128)
        _check(lib().ks_quad_rhs_finish(self._h, _ptr(out), KS_MEM_HOST))
        return out

    def ultraweak(self, f, u0, device: int = 0):
        """assemble_ultraweak (assembly.cpp:572-640) -> (A, rhs): the system
        operator and the load vector of f plus the initial-datum term
        i (u0, B_jt(0) phi_js); final-condition trial space only (InvalidArgument
        otherwise, as the reference's invalid_argument). u0: vectorised callable
        u0(x_1, .., x_d), sampled on the spatial quadrature grid."""
        if self.prob.trial != "final":
            raise InvalidArgument("assemble_ultraweak: problem must use the final-condition space")
        A = assemble_system_operator(self.prob, device=device)
        rhs = np.ascontiguousarray(self.assemble_rhs(f))
        u0s = self._sample(lambda *x: u0(*x), self.nodes[1:])
        _check(lib().ks_quad_initial_term(self._h, _ptr(u0s), KS_MEM_HOST, _ptr(rhs), KS_MEM_HOST))
        return A, rhs

    def lift(self, g, f):
        """lift_nonhomogeneous: (corrected rhs, boundary coefficients on the full space)."""
        rhs = self.assemble_rhs(f)
        bnd = np.zeros(self.N_full, dtype=np.complex128)
        corr = np.zeros(self.prob.N_dof, dtype=np.complex128)
        if isinstance(g, str):
            gd = DeviceVector(self.N_full)
            _check(lib().ks_quad_sample_named(self._h, g.encode(), 0, 1, 0, 0, gd.ptr))
            bd, cd = DeviceVector(self.N_full), DeviceVector(self.prob.N_dof)
            _check(lib().ks_quad_lift(self._h, gd.ptr, KS_MEM_DEVICE, bd.ptr, cd.ptr))
            bnd, corr = bd.to_host(), cd.to_host()
        else:
            gs = self._sample(g, self.greville)
            _check(lib().ks_quad_lift(self._h, _ptr(gs), KS_MEM_HOST, _ptr(bnd), _ptr(corr)))
        return rhs - corr, bnd

    def extend(self, reduced, boundary=None) -> np.ndarray:
        if isinstance(reduced, DeviceVector):
            reduced = reduced.to_host()
        reduced = _cvec(reduced).ravel()
        out = np.zeros(self.N_full, dtype=np.complex128)
        b = None if boundary is None else _cvec(boundary).ravel()
        _check(lib().ks_quad_extend(self._h, _ptr(reduced), None if b is None else _ptr(b), KS_MEM_HOST,
                                    _ptr(out)))
        return out

    def error_norms(self, full_coeffs, u, f):
        """(L2 error, sqrt(L2^2 + ||f - S u_h||^2)) as error_norms returns."""
        if isinstance(full_coeffs, DeviceVector):
            _check(lib().ks_quad_error_set(self._h, full_coeffs.ptr, KS_MEM_DEVICE))
        else:
            c = _cvec(full_coeffs).ravel()
            _check(lib().ks_quad_error_set(self._h, _ptr(c), KS_MEM_HOST))
        l2 = res = 0.0
        for r0, r1 in self._chunks():
            a, b = C.c_double(), C.c_double()
            if isinstance(u, str):
                bu, bf = self._chunk_buf()
                _check(lib().ks_quad_sample_named(self._h, u.encode(), 0, 0, r0, r1, bu.ptr))
                _check(lib().ks_quad_sample_named(self._h, u.encode(), 1, 0, r0, r1, bf.ptr))
                _check(lib().ks_quad_error_chunk(self._h, r0, r1, bu.ptr, bf.ptr, KS_MEM_DEVICE, C.byref(a),
                                                 C.byref(b)))
            else:
                coords = self.nodes[:self.d] + [self.nodes[self.d][r0:r1]]
                us, fs = self._sample(u, coords), self._sample(f, coords)
                _check(lib().ks_quad_error_chunk(self._h, r0, r1, _ptr(us), _ptr(fs), KS_MEM_HOST, C.byref(a),
                                                 C.byref(b)))
            l2 += a.value
            res += b.value
        return float(np.sqrt(l2)), float(np.sqrt(l2 + res))

    def __del__(self):
        try:
            if self._h:
                lib().ks_quad_destroy(self._h)
                self._h = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# PCG
# ---------------------------------------------------------------------------
@dataclass
class PcgOptions:
    tol: float = 1e-8
    maxit: int = 200
    strict_residual: bool = False


@dataclass
class SolveReport:
    x: np.ndarray
    iterations: int = 0
    res_history: List[float] = field(default_factory=list)
    converged: bool = False
    breakdown: bool = False
    restarts: int = 0
    setup_seconds: float = 0.0
    matvec_seconds: float = 0.0
    precond_seconds: float = 0.0
    solve_seconds: float = 0.0


def pcg(A: KroneckerOperator, P: Optional[FDPreconditioner], b, opts: PcgOptions = PcgOptions(),
        x_out: Optional[DeviceVector] = None) -> SolveReport:
    """Preconditioned CG with a device-resident loop (krylov.cpp:24-114)."""
    A._build()
    o = ks_pcg_opts(float(opts.tol), int(opts.maxit), int(bool(opts.strict_residual)))
    rep = ks_pcg_report()
    cap = max(int(opts.maxit), 1)
    hist = np.zeros(cap)
    if isinstance(b, DeviceVector):
        x = _dev_pair(A.vec_size(), b, x_out, "pcg")
        _check(lib().ks_pcg(A._h, P._h if P is not None else None, b.ptr, x.ptr, KS_MEM_DEVICE,
                            C.byref(o), _ptr(hist), cap, C.byref(rep)))
        xr = x
    else:
        bb = _cvec(b).ravel()
        if bb.size != A.vec_size():
            raise InvalidArgument("pcg: rhs length mismatch")
        xr = np.zeros_like(bb)
        _check(lib().ks_pcg(A._h, P._h if P is not None else None, _ptr(bb), _ptr(xr),
                            KS_MEM_HOST, C.byref(o), _ptr(hist), cap, C.byref(rep)))
    return SolveReport(x=xr, iterations=rep.iterations,
                       res_history=list(hist[:rep.hist_len]), converged=bool(rep.converged),
                       breakdown=bool(rep.breakdown), restarts=rep.restarts,
                       matvec_seconds=rep.matvec_seconds, precond_seconds=rep.precond_seconds,
                       solve_seconds=rep.solve_seconds)


def fp64_peaks():
    a, b = C.c_double(), C.c_double()
    _check(lib().ks_fp64_peaks(C.byref(a), C.byref(b)))
    return a.value, b.value


def fp64_peak_mma16():
    a = C.c_double()
    _check(lib().ks_fp64_peak_mma16(C.byref(a)))
    return a.value


def fp64_peak_mixed():
    a = C.c_double()
    _check(lib().ks_fp64_peak_mixed(C.byref(a)))
    return a.value


def bw_fan(nin: int, nout: int, n: int) -> float:
    """Streaming HBM throughput (GB/s) reading `nin` and writing `nout` complex vectors of n entries."""
    g = C.c_double()
    _check(lib().ks_bw_fan(nin, nout, n, C.byref(g)))
    return g.value


def launch_count() -> int:
    return int(lib().ks_launch_count())


def reset_launch_count():
    lib().ks_launch_count_reset()
