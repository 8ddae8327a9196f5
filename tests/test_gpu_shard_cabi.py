"""Multi-GPU through the C-ABI (include/ks.h ks_comm_*,
ks_fdshard_apply, ks_kronshard_apply_comm, ks_pcg_sharded): NCCL lives inside
libks, so a C++ caller of the reference's solver (experiments.cpp:46-52 ->
krylov.cpp:24) can run the slab-sharded FD preconditioner, matvec and PCG.

tests/cpp/sharded_pcg_demo.cpp is such a caller: one process per rank, the
unique id passed through a file. It runs with as many ranks as the box has
GPUs (NCCL refuses two ranks on one device, and ranks whose kernels wait on
each other must not share a GPU), at least one -- the single-rank run still
exercises the grouped send / recv all-to-alls, the halo exchange and the
device all-reduces -- and compares with the unsharded ks_pcg."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from helpers import rel, maxrel, setup_arrays

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build_demo(tmp):
    exe = os.path.join(tmp, "sharded_pcg_demo")
    lib = os.path.join(ROOT, "paper_2311_18461_b200")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "sharded_pcg_demo.cpp"), "-L" + lib, "-lks",
                           "-Wl,-rpath," + lib, "-o", exe])
    return exe


@pytest.mark.parametrize("d,p,n_el", [(3, 2, 12), (2, 3, 20)])
def test_cpp_sharded_pcg_through_cabi(gpu, d, p, n_el):
    nranks = max(1, min(2, gpu.device_count()))
    with tempfile.TemporaryDirectory() as tmp:
        exe = _build_demo(tmp)
        idf = os.path.join(tmp, "nccl.id")
        procs = [subprocess.Popen([exe, str(d), str(p), str(n_el), str(nranks), str(r), str(r), idf],
                                  stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
                 for r in range(nranks)]
        outs = []
        for pr in procs:
            o, e = pr.communicate(timeout=300)
            assert pr.returncode == 0, e
            outs.append(json.loads(o.strip().splitlines()[-1]))
    its = {o["iterations"] for o in outs}
    assert len(its) == 1 and all(o["converged"] for o in outs)
    r0 = next(o for o in outs if o["rank"] == 0)
    print(outs)
    # sharded vs one-GPU: the all-reduced dots sum in a different order -> counts +-1
    assert abs(r0["iterations"] - r0["single_gpu_iterations"]) <= 1
    assert r0["rel_vs_single"] <= 1e-6
    assert r0["final_relres"] <= 1e-8


def test_fdshard_and_halo_apply_single_rank_comm(gpu, oracle):
    """ks_fdshard_apply / ks_kronshard_apply_comm over a one-rank NCCL
    communicator equal the unsharded FD apply and matvec."""
    import ctypes as C
    import torch  # noqa: F401  (PyTorch's NCCL loads first; libks then uses the same library)
    from paper_2311_18461_b200 import dist
    L = gpu.lib()
    a = setup_arrays(gpu, 3, 2, 10, 6)
    uid = (C.c_char * 128)()
    gpu._check(L.ks_comm_unique_id(uid))
    comm = C.c_void_p()
    gpu._check(L.ks_comm_create(1, 0, uid, 0, C.byref(comm)))
    try:
        S = dist.ShardedFDPreconditioner(a["dims"], 1.0, a["p"], a["U"], a["lam"], a["Lt"], a["Mt"], a["Wt"],
                                         nranks=1, rank=0, device=0)
        n = a["prob"].N_dof
        r = oracle.random_vec(n, 12)
        rd, zd = gpu.DeviceVector.from_host(r), gpu.DeviceVector(n)
        gpu._check(L.ks_fdshard_apply(S._h, comm, rd.ptr, zd.ptr, None))
        zf = gpu.FDPreconditioner(a["prob"]).apply(r)
        assert rel(zd.to_host(), zf) <= 1e-12 and maxrel(zd.to_host(), zf) <= 1e-12
        K = dist.ShardedKroneckerOperator(a["prob"], nranks=1, rank=0, device=0)
        yd = gpu.DeviceVector(n)
        gpu._check(L.ks_kronshard_apply_comm(K._h, comm, rd.ptr, yd.ptr, None))
        yf = gpu.assemble_system_operator(a["prob"]).apply(r)
        assert rel(yd.to_host(), yf) <= 1e-13
    finally:
        L.ks_comm_destroy(comm)
