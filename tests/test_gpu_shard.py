"""Sharded FD phases (csrc/ks_shard.cu) on ONE GPU with P virtual ranks: each
rank's handle runs its phases in turn and the all-to-alls are emulated by
host copies (no kernel ever waits on another rank). The gathered result must
match the single-GPU FD apply and the oracle."""
import ctypes as C

import numpy as np
import pytest

from helpers import setup_arrays, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P,d,p,n_el,n_el_t", [(2, 2, 3, 10, 9), (3, 3, 2, 8, 8), (4, 3, 4, 6, 5),
                                               (2, 3, 2, 64, 64)])
def test_virtual_ranks_match_single_gpu(gpu, oracle, P, d, p, n_el, n_el_t):
    from paper_2311_18461_b200.dist import shard_plan
    ks = gpu
    L = ks.lib()
    a = setup_arrays(ks, d, p, n_el, n_el_t)
    dims, nt = a["dims"], a["dims"][0]
    Np = int(np.prod(dims[1:d]))
    N = int(np.prod(dims))
    r = oracle.random_vec(N, 1234)
    single = ks.FDPreconditioner.from_arrays(dims, 1.0, p, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
    z_ref = single.apply(r)
    d_ = len(dims) - 1
    Us = [np.ascontiguousarray(u).ravel() for u in a["U"]]
    ls = [np.ascontiguousarray(v).ravel() for v in a["lam"]]
    up = (C.c_void_p * d_)(*[x.ctypes.data for x in Us])
    lp = (C.c_void_p * d_)(*[x.ctypes.data for x in ls])
    cd = (C.c_int * (d_ + 1))(*dims)
    plans = [shard_plan(d_, dims, P, k) for k in range(P)]
    hs = []
    for k in range(P):
        h = C.c_void_p()
        ks._check(L.ks_fdshard_create(d_, cd, 1.0, p, up, lp, ks._ptr(a["Lt"]), ks._ptr(a["Mt"]),
                                      ks._ptr(a["Wt"]), P, k, 0, C.byref(h)))
        hs.append(h)
    # phase 1
    sends = []
    for k in range(P):
        lo, hi = plans[k]["slab"]
        rs = ks.DeviceVector.from_host(r[lo * nt * Np: hi * nt * Np])
        sb = ks.DeviceVector(max(sum(plans[k]["send_counts"]), 1))
        ks._check(L.ks_fdshard_forward(hs[k], rs.ptr, sb.ptr, None))
        sends.append(sb.to_host()[:sum(plans[k]["send_counts"])])
    # all-to-all #1 (emulated): rank q receives block q of every sender, in rank order
    works = []
    for q in range(P):
        parts = [sends[k][plans[k]["send_displs"][q]: plans[k]["send_displs"][q] + plans[k]["send_counts"][q]]
                 for k in range(P)]
        w = ks.DeviceVector.from_host(np.concatenate(parts))
        ks._check(L.ks_fdshard_middle(hs[q], w.ptr, None))
        works.append(w.to_host())
    # all-to-all #2: rank k receives from q the rows of its slab
    zs = []
    for k in range(P):
        parts = [works[q][plans[q]["recv_displs"][k]: plans[q]["recv_displs"][k] + plans[q]["recv_counts"][k]]
                 for q in range(P)]
        bk = ks.DeviceVector.from_host(np.concatenate(parts))
        lo, hi = plans[k]["slab"]
        zk = ks.DeviceVector((hi - lo) * nt * Np)
        ks._check(L.ks_fdshard_backward(hs[k], bk.ptr, zk.ptr, None))
        zs.append(zk.to_host())
    z = np.concatenate(zs)
    for h in hs:
        L.ks_fdshard_destroy(h)
    assert rel(z, z_ref) < 1e-12
    if N <= 400000:
        F = oracle.OracleFD(dims, 1.0, p, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
        assert rel(z, F.apply(r)) < 1e-10


def test_sharded_class_single_rank_nccl(gpu, oracle):
    """dist.ShardedFDPreconditioner end to end over a 1-rank NCCL group."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2311_18461_b200.dist import ShardedFDPreconditioner
    ks = gpu
    a = setup_arrays(ks, 3, 2, 10, 9)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        S = ShardedFDPreconditioner(a["dims"], 1.0, 2, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
        r = oracle.random_vec(int(np.prod(a["dims"])), 7)
        z = S.apply(torch.from_numpy(r).cuda()).cpu().numpy()
        torch.cuda.synchronize()
        single = ks.FDPreconditioner.from_arrays(a["dims"], 1.0, 2, a["U"], a["lam"], a["Lt"],
                                                 a["Mt"], a["Wt"])
        assert rel(z, single.apply(r)) < 1e-12
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,d,p,n_el", [(2, 2, 3, 10), (3, 3, 2, 8), (4, 3, 4, 16)])
def test_sharded_matvec_virtual_ranks(gpu, oracle, P, d, p, n_el):
    ks = gpu
    L = ks.lib()
    prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el)
    dims = prob.reduced_dims()
    plane = int(np.prod(dims[:d]))
    A = ks.assemble_system_operator(prob)
    x = oracle.random_vec(prob.N_dof, 5)
    y_ref = A.apply(x)
    ys = []
    for k in range(P):
        h = C.c_void_p()
        ks._check(L.ks_setup_create_system_sharded(prob._h, P, k, 0, C.byref(h)))
        lo, hi, elo, ehi = (C.c_longlong() for _ in range(4))
        pl = C.c_size_t()
        ks._check(L.ks_kronshard_sizes(h, C.byref(lo), C.byref(hi), C.byref(elo), C.byref(ehi), C.byref(pl)))
        assert pl.value == plane
        xe = ks.DeviceVector.from_host(x[elo.value * plane: ehi.value * plane])  # emulated halo exchange
        yk = ks.DeviceVector((hi.value - lo.value) * plane)
        ks._check(L.ks_kronshard_apply(h, xe.ptr, yk.ptr, None))
        ys.append(yk.to_host())
        L.ks_kron_destroy(h)
    assert rel(np.concatenate(ys), y_ref) < 1e-13


def test_sharded_pcg_single_rank_nccl(gpu, oracle):
    """dist.sharded_pcg with the sharded operators over a 1-rank NCCL group
    matches the device-resident ks_pcg."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2311_18461_b200.dist import (ShardedFDPreconditioner, ShardedKroneckerOperator,
                                            sharded_pcg)
    ks = gpu
    a = setup_arrays(ks, 3, 2, 12, 12)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        S = ShardedFDPreconditioner(a["dims"], 1.0, 2, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
        A = ShardedKroneckerOperator(a["prob"])
        b = oracle.random_vec(int(np.prod(a["dims"])), 1234)
        rep = sharded_pcg(A.apply, S.apply, torch.from_numpy(b).cuda())
        ref = ks.pcg(ks.assemble_system_operator(a["prob"]), ks.FDPreconditioner(a["prob"]), b)
        assert rep["converged"] and abs(rep["iterations"] - ref.iterations) <= 1
        assert rel(rep["x"].cpu().numpy(), ref.x) < 1e-7
    finally:
        dist.destroy_process_group()
