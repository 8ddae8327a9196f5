"""Multi-GPU slab-sharded FD preconditioner.

One process per GPU; the outermost spatial axis d is split in contiguous
slabs (`shard_plan`), so rank k owns the contiguous chunk
[slab_lo, slab_hi) x (n_t * N') of every vector in the reference's vec order.
`ShardedFDPreconditioner.apply` runs the three device phases of
`ks_fdshard_*` (csrc/ks_shard.cu) around two NCCL all-to-alls
(torch.distributed, backend "nccl"):

    forward (local transforms, pack) -> all_to_all -> middle (axis-d transform,
    block solves, inverse) -> all_to_all -> backward (unpack, inverse transforms)

Buffers are torch CUDA tensors; libks runs on torch's current stream, so the
collectives and kernels are stream-ordered without host syncs.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _check, _cvec, _ptr, lib
from . import ks_c64 as _C64


def shard_plan(d: int, dims: Sequence[int], nranks: int, rank: int) -> dict:
    """Host-only partition of axis d and the all-to-all counts (complex elements)."""
    LL = C.c_longlong
    lo, hi = LL(), LL()
    sc, sd, rc, rd = [(LL * nranks)() for _ in range(4)]
    cd = (C.c_int * (d + 1))(*dims)
    _check(lib().ks_shard_plan(d, cd, nranks, rank, C.byref(lo), C.byref(hi), sc, sd, rc, rd))
    return {"slab": (lo.value, hi.value), "send_counts": list(sc), "send_displs": list(sd),
            "recv_counts": list(rc), "recv_displs": list(rd)}


def _all_to_all_nccl(out, inp, out_counts, in_counts):
    import torch
    import torch.distributed as dist
    # complex128 as float64 pairs (NCCL reduces nothing here; it only moves bytes)
    dist.all_to_all_single(torch.view_as_real(out).reshape(-1), torch.view_as_real(inp).reshape(-1),
                           output_split_sizes=[2 * int(c) for c in out_counts],
                           input_split_sizes=[2 * int(c) for c in in_counts])


class ShardedFDPreconditioner:
    """FD preconditioner over `nranks` GPUs (one rank per process)."""

    def __init__(self, dims: Sequence[int], nu: float, p_t: int, U, lam, Lt, Mt, Wt,
                 nranks: Optional[int] = None, rank: Optional[int] = None, device: int = 0,
                 all_to_all: Optional[Callable] = None):
        import torch
        if nranks is None or rank is None:
            import torch.distributed as dist
            nranks, rank = dist.get_world_size(), dist.get_rank()
        self.dims, self.nranks, self.rank, self.device = list(dims), nranks, rank, device
        d = len(dims) - 1
        self.plan = shard_plan(d, dims, nranks, rank)
        Us = [np.ascontiguousarray(u, dtype=np.float64).ravel() for u in U]
        ls = [np.ascontiguousarray(v, dtype=np.float64).ravel() for v in lam]
        Lt = np.ascontiguousarray(Lt, dtype=np.float64).ravel()
        Mt = np.ascontiguousarray(Mt, dtype=np.float64).ravel()
        Wt = _cvec(Wt).ravel()
        up = (C.c_void_p * d)(*[a.ctypes.data for a in Us])
        lp = (C.c_void_p * d)(*[a.ctypes.data for a in ls])
        cd = (C.c_int * (d + 1))(*dims)
        h = C.c_void_p()
        _check(lib().ks_fdshard_create(d, cd, float(nu), int(p_t), up, lp, _ptr(Lt), _ptr(Mt),
                                       _ptr(Wt), nranks, rank, device, C.byref(h)))
        self._h = h
        sn, wn = C.c_size_t(), C.c_size_t()
        _check(lib().ks_fdshard_sizes(h, C.byref(sn), C.byref(wn)))
        self.slab_n, self.work_n = sn.value, wn.value
        dev = torch.device("cuda", device)
        self._send = torch.empty(sum(self.plan["send_counts"]), dtype=torch.complex128, device=dev)
        self._work = torch.empty(self.work_n, dtype=torch.complex128, device=dev)
        self._back = torch.empty(sum(self.plan["send_counts"]), dtype=torch.complex128, device=dev)
        self._a2a = all_to_all or _all_to_all_nccl

    def apply(self, r_slab, z_slab=None):
        """z_slab = (P^-1 r)[slab] for the local slab (torch complex128 CUDA tensors)."""
        import torch
        if z_slab is None:
            z_slab = torch.empty_like(r_slab)
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        L = lib()
        _check(L.ks_fdshard_forward(self._h, C.c_void_p(r_slab.data_ptr()),
                                    C.c_void_p(self._send.data_ptr()), st))
        self._a2a(self._work, self._send, self.plan["recv_counts"], self.plan["send_counts"])
        _check(L.ks_fdshard_middle(self._h, C.c_void_p(self._work.data_ptr()), st))
        self._a2a(self._back, self._work, self.plan["send_counts"], self.plan["recv_counts"])
        _check(L.ks_fdshard_backward(self._h, C.c_void_p(self._back.data_ptr()),
                                     C.c_void_p(z_slab.data_ptr()), st))
        return z_slab

    def __del__(self):
        try:
            if self._h:
                lib().ks_fdshard_destroy(self._h)
                self._h = None
        except Exception:
            pass


class PeerShardedFDPreconditioner(ShardedFDPreconditioner):
    """Sharded FD apply without all-to-alls: the middle phase's axis-d transform
    reads its rows straight from every rank's exported slab and its inverse
    writes them straight into every rank's output slab (peer memory over
    NVLink; CUDA IPC handles exchanged once through torch.distributed). Two
    barriers per apply separate the phases.

    For tests, `peers=(ins, outs)` (lists of tensors, one per rank, all in this
    process) replaces the IPC exchange and `barrier` the process group barrier."""

    def __init__(self, *args, peers=None, barrier=None, **kw):
        from . import DeviceVector
        super().__init__(*args, **kw)
        self._opened = []
        if peers is None:
            import torch.distributed as dist
            L = lib()
            # exported buffers from cudaMalloc directly: an IPC handle names the
            # whole allocation, so the buffers must start at their allocation base
            self._vin, self._vout = DeviceVector(self.slab_n), DeviceVector(self.slab_n)
            self.in_ptr, self.out_ptr = self._vin.ptr.value, self._vout.ptr.value
            hs = []
            for ptr in (self.in_ptr, self.out_ptr):
                buf = (C.c_char * 64)()
                _check(L.ks_ipc_get_handle(C.c_void_p(ptr), buf))
                hs.append(bytes(buf))
            allh = [None] * self.nranks
            dist.all_gather_object(allh, hs)
            ins, outs = [], []
            for q, (hi, ho) in enumerate(allh):
                if q == self.rank:
                    ins.append(self.in_ptr)
                    outs.append(self.out_ptr)
                    continue
                for hnd, dst in ((hi, ins), (ho, outs)):
                    ptr = C.c_void_p()
                    _check(L.ks_ipc_open(C.create_string_buffer(hnd, 64), C.byref(ptr)))
                    self._opened.append(ptr)
                    dst.append(ptr.value)
            self._barrier = barrier or (lambda: dist.barrier())
        else:
            ins = [t.data_ptr() for t in peers[0]]
            outs = [t.data_ptr() for t in peers[1]]
            self.in_ptr, self.out_ptr = ins[self.rank], outs[self.rank]
            self._barrier = barrier or (lambda: None)
        pin = (C.c_void_p * self.nranks)(*ins)
        pout = (C.c_void_p * self.nranks)(*outs)
        _check(lib().ks_fdshard_set_peers(self._h, pin, pout))

    def forward_slab(self, r_slab):
        import torch
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().ks_fdshard_forward_slab(self._h, C.c_void_p(r_slab.data_ptr()),
                                             C.c_void_p(self.in_ptr), st))

    def middle(self):
        import torch
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().ks_fdshard_middle_peer(self._h, st))

    def backward_slab(self, z_slab):
        import torch
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().ks_fdshard_backward_slab(self._h, C.c_void_p(self.out_ptr),
                                              C.c_void_p(z_slab.data_ptr()), st))

    def apply(self, r_slab, z_slab=None):
        import torch
        if z_slab is None:
            z_slab = torch.empty_like(r_slab)
        self.forward_slab(r_slab)
        torch.cuda.current_stream(self.device).synchronize()
        self._barrier()  # every rank's phase-1 slab is written
        self.middle()
        torch.cuda.current_stream(self.device).synchronize()
        self._barrier()  # every rank's output slab is complete
        self.backward_slab(z_slab)
        return z_slab

    def __del__(self):
        try:
            for ptr in self._opened:
                lib().ks_ipc_close(ptr)
            self._opened = []
        except Exception:
            pass
        super().__del__()


# ---------------------------------------------------------------------------
# sharded Kronecker-sum matvec: halo exchange of bw planes with the neighbours
# ---------------------------------------------------------------------------
def kron_shard_plan(n_d: int, bw: int, nranks: int, rank: int):
    """Host-only: owned planes [lo, hi) and haloed input [ext_lo, ext_hi) of a rank."""
    LL = C.c_longlong
    v = [LL() for _ in range(4)]
    _check(lib().ks_kronshard_plan(n_d, bw, nranks, rank, *[C.byref(x) for x in v]))
    return tuple(x.value for x in v)


def halo_exchange(ext, slab, plane, lo, hi, ext_lo, ext_hi, rank, nranks, send, recv):
    """Fill ext = [halo_lo | slab | halo_hi] from the neighbours: rank-1 sends its
    last (lo - ext_lo) planes, rank+1 its first (ext_hi - hi) planes; we send
    them the planes their halos need (bw each, the same width on both sides of
    an interior boundary). send/recv are point-to-point callables
    (tensor, peer) -> request-like; the default is NCCL via torch.distributed."""
    n_lo, n_hi = lo - ext_lo, ext_hi - hi
    bw = max(n_lo, n_hi)
    reqs = []
    if rank > 0:
        reqs.append(recv(ext[:n_lo * plane], rank - 1))
        reqs.append(send(slab[:bw * plane].contiguous(), rank - 1))
    if rank < nranks - 1:
        reqs.append(recv(ext[ext.numel() - n_hi * plane:], rank + 1))
        reqs.append(send(slab[slab.numel() - bw * plane:].contiguous(), rank + 1))
    for r in reqs:
        if r is not None:
            r.wait()


def _nccl_p2p():
    import torch.distributed as dist
    return (lambda t, peer: dist.isend(t, peer)), (lambda t, peer: dist.irecv(t, peer))


class ShardedKroneckerOperator:
    """The system operator A (assembly.cpp:202-251) slab-sharded like the FD
    preconditioner: apply(x_slab) -> y_slab after a halo exchange."""

    def __init__(self, prob, nranks: Optional[int] = None, rank: Optional[int] = None,
                 device: int = 0, halo: Optional[Callable] = None):
        import torch
        if nranks is None or rank is None:
            import torch.distributed as dist
            nranks, rank = dist.get_world_size(), dist.get_rank()
        self.nranks, self.rank, self.device = nranks, rank, device
        h = C.c_void_p()
        _check(lib().ks_setup_create_system_sharded(prob._h, nranks, rank, device, C.byref(h)))
        self._h = h
        lo, hi, elo, ehi = (C.c_longlong() for _ in range(4))
        plane = C.c_size_t()
        _check(lib().ks_kronshard_sizes(h, C.byref(lo), C.byref(hi), C.byref(elo), C.byref(ehi),
                                        C.byref(plane)))
        self.lo, self.hi, self.ext_lo, self.ext_hi = lo.value, hi.value, elo.value, ehi.value
        self.plane = plane.value
        self.n_lo, self.n_hi = self.lo - self.ext_lo, self.ext_hi - self.hi
        self._ext = torch.empty((self.ext_hi - self.ext_lo) * self.plane, dtype=torch.complex128,
                                device=torch.device("cuda", device))
        self._halo = halo

    def apply(self, x_slab, y_slab=None):
        import torch
        if y_slab is None:
            y_slab = torch.empty_like(x_slab)
        a, b = self.n_lo * self.plane, self.n_lo * self.plane + x_slab.numel()
        self._ext[a:b].copy_(x_slab)
        send, recv = self._halo if self._halo is not None else _nccl_p2p()
        halo_exchange(self._ext, x_slab, self.plane, self.lo, self.hi, self.ext_lo, self.ext_hi,
                      self.rank, self.nranks, send, recv)
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().ks_kronshard_apply(self._h, C.c_void_p(self._ext.data_ptr()),
                                        C.c_void_p(y_slab.data_ptr()), st))
        return y_slab

    def __del__(self):
        try:
            if self._h:
                lib().ks_kron_destroy(self._h)
                self._h = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# sharded PCG: krylov.cpp:24-114 control flow, local BLAS-1 in libks, global
# sums by all-reduce
# ---------------------------------------------------------------------------
def sharded_pcg(apply_a, apply_p, b_slab, tol=1e-8, maxit=200, strict=False, allreduce=None):
    """PCG over slab-sharded vectors. apply_a / apply_p map a torch slab to a
    torch slab (the sharded operators); allreduce sums a python float over ranks
    (default: torch.distributed NCCL)."""
    import torch
    if allreduce is None:
        import torch.distributed as dist

        def allreduce(v):
            t = torch.tensor([v], dtype=torch.float64, device=b_slab.device)
            dist.all_reduce(t)
            return float(t.item())
    if not (tol > 0) or maxit < 0:
        raise ValueError("pcg: bad options")
    L = lib()
    n = b_slab.numel()
    st = C.c_void_p(torch.cuda.current_stream(b_slab.device).cuda_stream)
    ptr = lambda t: C.c_void_p(t.data_ptr())

    def dot_re(x, y):
        out = _C64()
        torch.cuda.synchronize(b_slab.device)
        _check(L.ks_dotc(ptr(x), ptr(y), n, C.byref(out), st))
        return allreduce(out.re)

    def norm2(x):
        v = C.c_double()
        torch.cuda.synchronize(b_slab.device)
        _check(L.ks_norm2sq(ptr(x), n, C.byref(v), st))
        return allreduce(v.value)

    x = torch.zeros_like(b_slab)
    hist = []
    bnorm = norm2(b_slab) ** 0.5
    rep = {"x": x, "iterations": 0, "res_history": hist, "converged": False, "breakdown": False}
    if bnorm == 0.0:
        rep["converged"] = True
        return rep

    def true_relres():
        s = apply_a(x)
        s.sub_(b_slab)
        return norm2(s) ** 0.5 / bnorm, s

    r = b_slab.clone()
    z = apply_p(r) if apply_p else r.clone()
    p = z.clone()
    rho = dot_re(r, z)
    restarts = 0
    for _ in range(maxit):
        q = apply_a(p)
        curv = dot_re(p, q)
        if curv <= 0.0:
            rep["breakdown"] = True
            break
        alpha = rho / curv
        rr = C.c_double()
        torch.cuda.synchronize(b_slab.device)
        _check(L.ks_cg_update(alpha, ptr(p), ptr(q), ptr(x), ptr(r), n, C.byref(rr), st))
        rep["iterations"] += 1
        relres = allreduce(rr.value) ** 0.5 / bnorm
        if strict:
            relres, _ = true_relres()
        hist.append(relres)
        if relres <= tol:
            if not strict:
                tr, s = true_relres()
                hist[-1] = tr
                if tr > tol:
                    restarts += 1
                    if restarts > 2:
                        break
                    r = -s
                    z = apply_p(r) if apply_p else r.clone()
                    p = z.clone()
                    rho = dot_re(r, z)
                    continue
            rep["converged"] = True
            break
        z = apply_p(r) if apply_p else r.clone()
        rho_new = dot_re(r, z)
        beta = rho_new / rho
        rho = rho_new
        torch.cuda.synchronize(b_slab.device)
        _check(L.ks_xpby(ptr(z), beta, ptr(p), n, st))
    return rep
