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
