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


@pytest.mark.parametrize("P,d,p,n_el,n_el_t", [(2, 2, 3, 10, 9), (3, 3, 2, 8, 8), (4, 3, 4, 6, 5),
                                               (2, 3, 2, 64, 64)])
def test_peer_transport_virtual_ranks(gpu, oracle, P, d, p, n_el, n_el_t):
    """Peer-memory transport (ks_fdshard_*_slab / _middle_peer): P virtual ranks
    in this process export their slabs as plain device pointers; the middle
    phase gathers / scatters the axis-d rows straight from / into the other
    ranks' slabs. Phases run rank by rank (the barrier is the phase order)."""
    import torch
    from paper_2311_18461_b200.dist import PeerShardedFDPreconditioner
    ks = gpu
    a = setup_arrays(ks, d, p, n_el, n_el_t)
    dims, nt = a["dims"], a["dims"][0]
    Np = int(np.prod(dims[1:d]))
    N = int(np.prod(dims))
    r = oracle.random_vec(N, 99)
    z_ref = ks.FDPreconditioner.from_arrays(dims, 1.0, p, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"]).apply(r)
    from paper_2311_18461_b200.dist import shard_plan
    plans = [shard_plan(d, dims, P, k) for k in range(P)]
    sizes = [(pl["slab"][1] - pl["slab"][0]) * nt * Np for pl in plans]
    ins = [torch.empty(n, dtype=torch.complex128, device="cuda") for n in sizes]
    outs = [torch.empty(n, dtype=torch.complex128, device="cuda") for n in sizes]
    ranks = []
    for k in range(P):
        S = PeerShardedFDPreconditioner(dims, 1.0, p, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"],
                                        nranks=P, rank=k, device=0, peers=(ins, outs))
        ranks.append(S)
    rt = torch.from_numpy(r).cuda()
    for k, S in enumerate(ranks):
        lo, hi = plans[k]["slab"]
        S.forward_slab(rt[lo * nt * Np: hi * nt * Np])
    torch.cuda.synchronize()
    for S in ranks:
        S.middle()
    torch.cuda.synchronize()
    zs = []
    for k, S in enumerate(ranks):
        zk = torch.empty(sizes[k], dtype=torch.complex128, device="cuda")
        S.backward_slab(zk)
        zs.append(zk)
    torch.cuda.synchronize()
    z = torch.cat(zs).cpu().numpy()
    assert rel(z, z_ref) < 1e-12


def _ipc_worker(rank, ws, port, q):
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    try:
        import torch
        import torch.distributed as dist
        import paper_2311_18461_b200 as ks
        from paper_2311_18461_b200.dist import PeerShardedFDPreconditioner, shard_plan
        from oracle import oracle as O
        from helpers import setup_arrays
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        d, p = 3, 2
        a = setup_arrays(ks, d, p, 12, 10)
        dims, nt = a["dims"], a["dims"][0]
        Np = int(np.prod(dims[1:d]))
        r = O.random_vec(int(np.prod(dims)), 5)
        S = PeerShardedFDPreconditioner(dims, 1.0, p, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"],
                                        nranks=ws, rank=rank, device=0)
        lo, hi = shard_plan(d, dims, ws, rank)["slab"]
        zk = S.apply(torch.from_numpy(r[lo * nt * Np: hi * nt * Np].copy()).cuda())
        torch.cuda.synchronize()
        parts = [None] * ws
        dist.all_gather_object(parts, zk.cpu().numpy())
        if rank == 0:
            z = np.concatenate(parts)
            zr = ks.FDPreconditioner.from_arrays(dims, 1.0, p, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"]).apply(r)
            q.put(float(np.linalg.norm(z - zr) / np.linalg.norm(zr)))
        dist.barrier()
        del S
        dist.destroy_process_group()
    except Exception as e:
        q.put(repr(e))
        raise


def test_peer_transport_cuda_ipc_two_processes(gpu):
    """The same peer transport across two processes through CUDA IPC handles
    (exchanged with all_gather_object; gloo barriers between the phases). Both
    processes share the one GPU of the test box; no kernel waits on the other
    process -- the host barriers order the phases."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(k, 2, port, q)) for k in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    res = q.get(timeout=10)
    assert not isinstance(res, str), res
    assert res < 1e-12
