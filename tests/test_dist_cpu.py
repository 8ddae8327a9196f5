"""Multi-rank host logic of the slab-sharded FD preconditioner on the CPU
(gloo, world_size 2 and 3): the partition and all-to-all counts come from
libks (ks_shard_plan, host-only); the three device phases of csrc/ks_shard.cu
are restated here in numpy (same pack/unpack layout, same fiber -> block
mapping by global spatial index) with the oracle's banded solves, and the
gathered result must equal the oracle's single-process FD application."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, d, p, n_el, n_el_t, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    import paper_2311_18461_b200 as ks
    from paper_2311_18461_b200.dist import shard_plan
    from oracle import oracle as O
    from helpers import setup_arrays
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        a = setup_arrays(ks, d, p, n_el, n_el_t)
        dims, nt = a["dims"], a["dims"][0]
        Np = int(np.prod(dims[1:d]))
        plan = shard_plan(d, dims, ws, rank)
        lo, hi = plan["slab"]
        m = hi - lo
        F = O.OracleFD(dims, 1.0, p, a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"])
        r = O.random_vec(F.N, 1234)
        r_slab = r[lo * nt * Np: hi * nt * Np]
        Um = [a["U"][l].reshape(dims[l + 1], dims[l + 1]).T for l in range(d)]  # Um[j, r] = U(j, r)

        def ax_of(l, ndim):  # numpy axis of spatial axis l (1-based) in a reversed-shape array
            return ndim - 1 - l

        # forward: transforms U^T on axes 1..d-1 of the slab
        X = r_slab.reshape([m] + [dims[l] for l in range(d - 1, 0, -1)] + [nt])
        for l in range(1, d):
            ax = ax_of(l, X.ndim)
            X = np.moveaxis(np.tensordot(Um[l - 1].T, X, axes=([1], [ax])), 0, ax)
        X3 = X.reshape(m, Np, nt)
        # rest ranges reproduced from the plan's counts: send_counts[q] = nt * |R_q| * m
        Rn = [c // (nt * m) if m else 0 for c in plan["send_counts"]]
        Rlo = np.cumsum([0] + Rn[:-1])
        send = np.concatenate([X3[:, Rlo[k]:Rlo[k] + Rn[k], :].ravel() for k in range(ws)])
        assert send.size == sum(plan["send_counts"])
        work = np.empty(sum(plan["recv_counts"]), dtype=np.complex128)
        dist.all_to_all_single(torch.from_numpy(work.view(np.float64)),
                               torch.from_numpy(send.view(np.float64)),
                               output_split_sizes=[2 * c for c in plan["recv_counts"]],
                               input_split_sizes=[2 * c for c in plan["send_counts"]])
        # middle: (n_d, |R|, nt) -> axis-d transform, block solves, inverse transform
        Rme = Rn[rank]
        W = work.reshape(dims[d], Rme, nt)
        W = np.tensordot(Um[d - 1].T, W, axes=([1], [0]))
        for i_d in range(dims[d]):
            for rl in range(Rme):
                i = (Rlo[rank] + rl) + Np * i_d  # global spatial index (axis 1 fastest)
                ab, piv = F.block(i)
                x = np.ascontiguousarray(W[i_d, rl, :])
                O.olib().ko_solve_banded(O._p(ab), O._p(piv), nt, p, O._p(x))
                W[i_d, rl, :] = x
        W = np.tensordot(Um[d - 1], W, axes=([1], [0]))
        back_send = np.ascontiguousarray(W).ravel()
        back = np.empty(sum(plan["send_counts"]), dtype=np.complex128)
        dist.all_to_all_single(torch.from_numpy(back.view(np.float64)),
                               torch.from_numpy(back_send.view(np.float64)),
                               output_split_sizes=[2 * c for c in plan["send_counts"]],
                               input_split_sizes=[2 * c for c in plan["recv_counts"]])
        # backward: unpack, inverse transforms U on axes 1..d-1
        Y3 = np.empty((m, Np, nt), dtype=np.complex128)
        off = 0
        for k in range(ws):
            blk = back[off:off + plan["send_counts"][k]].reshape(m, Rn[k], nt)
            Y3[:, Rlo[k]:Rlo[k] + Rn[k], :] = blk
            off += plan["send_counts"][k]
        Y = Y3.reshape([m] + [dims[l] for l in range(d - 1, 0, -1)] + [nt])
        for l in range(1, d):
            ax = ax_of(l, Y.ndim)
            Y = np.moveaxis(np.tensordot(Um[l - 1], Y, axes=([1], [ax])), 0, ax)
        z_slab = Y.ravel()
        gathered = [None] * ws
        dist.all_gather_object(gathered, z_slab)
        if rank == 0:
            z = np.concatenate(gathered)
            zo = F.apply(r)
            q.put(float(np.linalg.norm(z - zo) / np.linalg.norm(zo)))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the test
        q.put(repr(e))
        raise


@pytest.mark.parametrize("ws,d,p,n_el,n_el_t", [(2, 2, 2, 6, 5), (2, 3, 2, 4, 4), (3, 3, 3, 5, 4)])
def test_sharded_fd_matches_oracle_gloo(ws, d, p, n_el, n_el_t):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, ws, port, d, p, n_el, n_el_t, q)) for k in range(ws)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    res = q.get(timeout=10)
    assert not isinstance(res, str), res
    assert res < 1e-12


def test_shard_plan_counts(ks):
    from paper_2311_18461_b200.dist import shard_plan
    dims = [131, 130, 130, 130]  # config 5: uneven slabs over 4 and 8 ranks
    for ws in (2, 4, 8):
        tot_send = 0
        for k in range(ws):
            pl = shard_plan(3, dims, ws, k)
            lo, hi = pl["slab"]
            assert hi - lo in (130 // ws, 130 // ws + 1)
            assert sum(pl["send_counts"]) == 131 * 130 * 130 * (hi - lo)
            assert pl["send_displs"][0] == 0 and pl["recv_displs"][0] == 0
            tot_send += sum(pl["send_counts"])
        assert tot_send == 131 * 130 ** 3
    with pytest.raises(ks.InvalidArgument):
        shard_plan(1, [66, 65], 2, 0)  # d = 1 cannot re-shard axes 1..d-1


def _halo_worker(rank, ws, port, d, p, n_el, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    import paper_2311_18461_b200 as ks
    from paper_2311_18461_b200.dist import kron_shard_plan, halo_exchange
    from oracle import oracle as O
    from helpers import setup_arrays
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=ws)
        a = setup_arrays(ks, d, p, n_el, n_el)
        dims = a["dims"]
        plane = int(np.prod(dims[:d]))
        lo, hi, elo, ehi = kron_shard_plan(dims[d], p, ws, rank)
        K = O.OracleKron(dims, O.system_terms(a, d, 1.0))
        x = O.random_vec(K.N, 99)
        xs = torch.from_numpy(x[lo * plane: hi * plane].copy())
        ext = torch.zeros((ehi - elo) * plane, dtype=torch.complex128)
        ext[(lo - elo) * plane:(lo - elo) * plane + xs.numel()] = xs
        send = lambda t, peer: dist.isend(torch.view_as_real(t).reshape(-1), peer)
        recv = lambda t, peer: _Recv(t, peer)
        halo_exchange(ext, xs, plane, lo, hi, elo, ehi, rank, ws, send, recv)
        # y[lo:hi] depends only on x[ext_lo:ext_hi] (banded outermost factors): zero elsewhere
        xg = np.zeros(K.N, dtype=np.complex128)
        xg[elo * plane: ehi * plane] = ext.numpy()
        y_slab = K.apply(xg)[lo * plane: hi * plane]
        gathered = [None] * ws
        dist.all_gather_object(gathered, y_slab)
        if rank == 0:
            y = np.concatenate(gathered)
            yo = K.apply(x)
            q.put(float(np.linalg.norm(y - yo) / np.linalg.norm(yo)))
        dist.destroy_process_group()
    except Exception as e:
        q.put(repr(e))
        raise


class _Recv:
    """gloo recv into a complex tensor view (irecv + copy back on wait)."""

    def __init__(self, t, peer):
        import torch.distributed as dist
        self.t = t
        self.buf = torch_view = __import__("torch").empty(t.numel() * 2, dtype=__import__("torch").float64)
        self.req = dist.irecv(torch_view, peer)

    def wait(self):
        import torch
        self.req.wait()
        self.t.copy_(torch.view_as_complex(self.buf.view(-1, 2)))


@pytest.mark.parametrize("ws,d,p,n_el", [(2, 2, 2, 8), (3, 3, 2, 6), (2, 3, 3, 6)])
def test_sharded_matvec_halo_gloo(ws, d, p, n_el):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(k, ws, port, d, p, n_el, q)) for k in range(ws)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    res = q.get(timeout=10)
    assert not isinstance(res, str), res
    assert res < 1e-14
