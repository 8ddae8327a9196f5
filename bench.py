#!/usr/bin/env python
"""Benchmark: FD preconditioner application DOF/s (complex FP64) on B200.

Headline workload (BASELINE.json configs[2], "c3"): d=3 space + time on
[0,1]^3 x [0,1], p=2, maximal regularity, 64 elements per direction,
reduced dims (65, 64, 64, 64) = 17,039,360 complex DOF; RHS re/im i.i.d.
U[-1,1] from seed 1234. configs[1] (d=2, 279K DOF) is latency-bound and is
reported as the full-solve leg ("solve_c2"); c3 is the largest single-GPU
config the metric's roofline target is quoted on.

A "step" is one FD preconditioner application over the whole c3 tensor with
the input resident in HBM. `value` = DOF/s over all ranks; `e2e` = the same
through the public host-pointer API (H2D of r and D2H of z inside the timed
region, pinned host memory). The tensor (272 MB) is larger than L2 (126 MB),
so no explicit flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (d, p, n_el, n_el_time)
    "c1": (1, 3, 64, 64),
    "c2": (2, 3, 64, 64),
    "c3": (3, 2, 64, 64),
    "c5": (3, 4, 128, 128),
}


def reduced_dims(cfg):
    """SpaceTimeProblem::uniform reduced dims (assembly.hpp:29-63, initial-condition
    trial space): n_t = n_el_t + p - 1, n_s = n_el + p - 2 -- no library needed."""
    d, p, n_el, n_el_t = CONFIGS[cfg]
    return [n_el_t + p - 1] + [n_el + p - 2] * d


def bench_config(cfg, ws):
    """The `config` object both arms print (identical dicts: the driver compares them)."""
    d, p, n_el, n_el_t = CONFIGS[cfg]
    dims = reduced_dims(cfg)
    n = int(np.prod(dims))
    return {"workload": f"{cfg}: d={d} p={p} n_el={n_el} n_el_t={n_el_t}, "
                        "one FD preconditioner application per step",
            "dims": dims, "dofs": n,
            "parallelism": "single" if ws == 1 else f"slab{ws} (outermost spatial axis)",
            "l2": (f"inputs ({n * 16 / 1e6:.0f} MB/vector) larger than the 126 MB L2; no flush"
                   if n * 16 > 126e6 else f"inputs ({n * 16 / 1e6:.1f} MB/vector) L2-resident (latency-bound size)")}


def fd_flops_per_dof(dims, p):
    # F_alg = 8 * sum_l n_l + 24 p + 8 (dense transforms + pivoted banded solve)
    return 8 * sum(dims[1:]) + 24 * p + 8


def fd_folded_flops_per_dof(dims, p, folded):
    """Flops of the transforms as executed: a folded axis does two (n/2 x n/2)
    products (4n flop/DOF for forward + inverse, plus 2 fold adds each way)."""
    t = sum((4 * dims[l] + 4) if l in folded else 8 * dims[l] for l in range(1, len(dims)))
    return t + 24 * p + 8


def matvec_flops_per_dof(d, p):
    return 24 * d * (2 * p + 1)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def ncu_traffic(kernel_substr):
    """DRAM bytes (read + write) per launch of a kernel from the newest committed
    `ncu --set full` summary (profiles/*/ncu_fd_matvec_metrics.csv, written by
    tools/ncu_summary.py), averaged over its launches; None if absent."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_fd_matvec_metrics.csv")))
    if not files:
        return None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        with open(files[-1]) as f:
            rows = list(csv.reader(f))
        h, u = rows[0], rows[1]
        ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
        vals = [float(r[ir]) * scale.get(u[ir], 1.0) + float(r[iw]) * scale.get(u[iw], 1.0)
                for r in rows[2:] if kernel_substr in r[ik]]
        return {"bytes_per_launch": sum(vals) / len(vals), "launches": len(vals),
                "source": os.path.relpath(files[-1], ROOT)} if vals else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        return rank, ws, local, dist
    return rank, ws, local, None


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rhs(n, seed=1234):
    """RHS re/im i.i.d. U[-1,1] (bench-side generator; the oracle has its own MT19937-64)."""
    g = np.random.default_rng(seed)
    v = np.empty(n, dtype=np.complex128)
    v.real = g.uniform(-1.0, 1.0, n)
    v.imag = g.uniform(-1.0, 1.0, n)
    return v


def _ref_apply(cfg):
    """The reference CPU FD application on the host: oracle/_ref (the reference's own
    sources, oracle/build_ref.sh) when built, else the C restatement (`kind` "port").
    Single-threaded, like the reference. Errors propagate."""
    d, p, n_el, n_el_t = CONFIGS[cfg]
    from oracle import refdrv
    if refdrv.available():
        ref = refdrv.RefProblem(d, p, n_el, n_el_t)
        return "reference", ref.fd_apply, ref.N
    # no reference build on this host (oracle/_ref is built by __graft_entry__.build()
    # and ships with the tree): the bit-exact C restatement (oracle/ks_oracle.c), fed
    # by libks's host-only setup restatement (pure host code, no device work)
    from oracle import oracle as O
    import paper_2311_18461_b200 as ks
    O.build_oracle()
    prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el_t)
    Lt, Mt, Wt = prob.time_bands()
    U, lam = zip(*[prob.eig(l) for l in range(d)])
    fd = O.OracleFD(prob.reduced_dims(), 1.0, p, U, lam, Lt, Mt, Wt)
    return "port", fd.apply, prob.N_dof


def cpu_baseline_fd(cfg, r, steps=3, warmup=1):
    """cpu_baseline leg: `warmup` excluded applications, then the
    median of `steps` timed ones (std::chrono-equivalent perf_counter around each)."""
    kind, apply, _ = _ref_apply(cfg)
    for _ in range(warmup):
        apply(r)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        apply(r)
        times.append(time.perf_counter() - t0)
    return kind, float(np.median(times)), len(times)


def _ref_worker(cfg, n, steps, warm, start, q):
    """One host core's share of the reference arm: its own reference problem (the
    reference is single-threaded, so independent applications are how it uses a
    multi-core host), `warm` untimed applications, then `steps` timed ones after
    the common start."""
    try:
        kind, apply, nref = _ref_apply(cfg)
        assert nref == n, (nref, n)
        r = rhs(n)
        for _ in range(warm):
            apply(r)
        start.wait()
        t0 = time.perf_counter()
        for _ in range(steps):
            apply(r)
        q.put((kind, steps, t0, time.perf_counter()))
    except BaseException as e:  # report instead of hanging the parent
        start.abort()
        q.put(("error", repr(e), 0.0, 0.0))


def ref_workers(K):
    """Concurrent reference processes: the largest divisor of K that the host's
    cores and free memory (~3 GB per c3 reference problem) can hold, so the K
    timed applications split evenly over them."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    try:
        import psutil
        mem = int(psutil.virtual_memory().available // (3 << 30))
    except Exception:
        mem = cores
    cap = int(os.environ.get("KS_REF_WORKERS", "0")) or max(1, min(cores, mem, 64))
    return max(w for w in range(1, min(cap, K) + 1) if K % w == 0)


def run_reference_arm(args, rank, ws, dist):
    """--impl reference: the reference's own CPU FD application (oracle/_ref) on the
    host cores, same config / metric / steps / warm-up as our arm. The K timed
    applications are spread evenly over concurrent single-threaded reference
    processes (the reference never threads); value = K x N_dof / concurrent wall
    time. libks is never loaded in this arm."""
    if rank != 0:
        return
    cfg = args.config
    n = int(np.prod(reduced_dims(cfg)))
    K = args.steps
    W = max(args.warmup, 3)
    workers = ref_workers(K)
    per = K // workers
    warm = -(-W // workers)  # every process warms up; >= W applications in total
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    start = ctx.Barrier(workers + 1)
    q = ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, args=(cfg, n, per, warm, start, q)) for _ in range(workers)]
    for pr in procs:
        pr.start()
    start.wait()
    res = [q.get() for _ in procs]
    for pr in procs:
        pr.join()
    bad = [x for x in res if x[0] == "error"]
    if bad:
        raise SystemExit(f"reference worker failed: {bad[0][1]}")
    kind = res[0][0]
    wall = max(x[3] for x in res) - min(x[2] for x in res)
    val = K * n / wall
    line = {
        "metric": "fd_apply_dof_per_s", "value": val, "unit": "DOF/s", "n_gpus": ws,
        "steps": K, "warmup": W, "ms_per_step": wall / K * 1e3,
        "higher_is_better": True, "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None,
        "dtype": "c128 (complex FP64)",
        "data": "synthetic (seeded U[-1,1] RHS, SURVEY 8(d))", "impl": "reference",
        "config": bench_config(cfg, ws),
        "cpu_baseline": {"value": val, "unit": "DOF/s", "cores": workers, "kind": kind,
                         "sample": f"{K} full {cfg} FD applications split over {workers} concurrent "
                                   f"single-threaded reference processes ({per} each, after "
                                   f"{warm} untimed each); value = K x N_dof / concurrent wall time"},
        "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, rank, ws, local, dist):
    """N > 1: the c3 problem slab-sharded over N GPUs (strong scaling). FD apply
    with the peer-memory transport (PeerShardedFDPreconditioner: the axis-d
    transform gathers / scatters its rows from / to the other GPUs' slabs over
    NVLink) when it reproduces the NCCL all-to-all version on this box, which is
    timed alongside (ShardedFDPreconditioner)."""
    import torch
    import paper_2311_18461_b200 as ks
    from paper_2311_18461_b200.dist import ShardedFDPreconditioner
    d, p, n_el, n_el_t = CONFIGS[args.config]
    W = max(args.warmup, 3)
    K = args.steps
    prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el_t)
    dims = prob.reduced_dims()
    n = prob.N_dof
    Lt, Mt, Wt = prob.time_bands()
    U, lam = zip(*[prob.eig(l) for l in range(d)])
    S_nccl = ShardedFDPreconditioner(dims, 1.0, p, U, lam, Lt, Mt, Wt, device=local)
    lo, hi = S_nccl.plan["slab"]
    per = dims[0] * int(np.prod(dims[1:d]))
    r_host = rhs(n)[lo * per: hi * per]
    r = torch.from_numpy(r_host).to(f"cuda:{local}")
    z = torch.empty_like(r)

    def time_fd(S):
        for _ in range(W):
            S.apply(r, z)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(K):
            S.apply(r, z)
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        return max_over_ranks(dist, e0.elapsed_time(e1) / K)

    # transport: peer memory (the axis-d transform reads / writes the other GPUs'
    # slabs over NVLink, no all-to-all) when it reproduces the NCCL result on
    # this box, else the NCCL all-to-all version
    transport, transport_note = args.transport, None
    z_ref = S_nccl.apply(r).clone()
    S = S_nccl
    if transport in ("auto", "peer"):
        S_peer, failed = None, 0.0
        try:
            from paper_2311_18461_b200.dist import PeerShardedFDPreconditioner
            S_peer = PeerShardedFDPreconditioner(dims, 1.0, p, U, lam, Lt, Mt, Wt, device=local)
        except Exception as e:  # no P2P / IPC on this box
            failed, transport_note = 1.0, f"peer transport unavailable: {e}"
        if max_over_ranks(dist, failed) > 0:  # every rank agrees before any peer phase runs
            transport = "nccl"
            transport_note = transport_note or "peer transport unavailable on another rank"
        else:
            zq = S_peer.apply(r)
            err = max_over_ranks(dist, float(torch.linalg.norm(zq - z_ref) / torch.linalg.norm(z_ref)))
            if err <= 1e-12:
                S, transport = S_peer, "peer"
            else:
                transport, transport_note = "nccl", f"peer transport mismatch {err:.2e}"
    ms_nccl = time_fd(S_nccl) if S is not S_nccl else None
    ks.reset_launch_count()
    clk = ClockSampler(local).__enter__()
    ms = time_fd(S)
    launches = ks.launch_count() // max(1, K + W)  # per apply (time_fd runs W + K)
    # e2e: host slab in (pinned), apply, host slab out, every step
    rp = torch.from_numpy(r_host).pin_memory()
    zp = torch.empty_like(rp).pin_memory()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(K):
        rd = rp.to(f"cuda:{local}", non_blocking=True)
        S.apply(rd, z)
        zp.copy_(z, non_blocking=True)
        torch.cuda.synchronize()
    e2e = (time.perf_counter() - t0) / K
    clk.__exit__(None, None, None)
    e2e = max_over_ranks(dist, e2e)
    # full sharded solve to 1e-8 (sharded matvec with halo exchange + sharded FD + all-reduce dots)
    solves = {}
    if not args.no_solve:
        from paper_2311_18461_b200.dist import ShardedKroneckerOperator, sharded_pcg
        A = ShardedKroneckerOperator(prob, device=local)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        rep = sharded_pcg(A.apply, S.apply, r, 1e-8, 200)
        torch.cuda.synchronize()
        sec = max_over_ranks(dist, time.perf_counter() - t0)
        solves[f"solve_{args.config}"] = {"iterations": rep["iterations"], "converged": rep["converged"],
                                          "seconds": sec,
                                          "final_relres": rep["res_history"][-1] if rep["res_history"] else None}
    # whole-job roofline of the sharded FD apply (SURVEY 8(d) dense F_alg, N x the
    # per-GPU FP64 peak measured live on every rank, the slowest rank's peak)
    ks.lib().ks_set_device(local)  # the library's own runtime: peak kernels on this rank's GPU
    dfma, dmma = ks.fp64_peaks()
    fp64_peak = max_over_ranks(dist, -max(dfma, dmma)) * -1.0
    hbm_peak = peaks().get("hbm_gbs", 6650.0)
    roof_s = max(fd_flops_per_dof(dims, p) * n / (ws * fp64_peak * 1e12), 32.0 * n / (ws * hbm_peak * 1e9))
    roofline = {"bound": "fp64", "achieved": fd_flops_per_dof(dims, p) * n / (ms * 1e-3) / 1e12,
                "peak": ws * fp64_peak, "unit": "TFLOP/s", "frac": roof_s / (ms * 1e-3), "traffic": None,
                "kernel": "whole sharded FD apply (all ranks)",
                "basis": "SURVEY 8(d) dense F_alg per DOF x N_dof per apply / max-over-ranks apply time; "
                         "peak = n_gpus x min-over-ranks live DFMA/DMMA peak"}
    if rank == 0:
        print(json.dumps({
            "metric": "fd_apply_dof_per_s", "value": n / (ms * 1e-3), "unit": "DOF/s", "n_gpus": ws,
            "steps": K, "warmup": W, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (complex FP64)",
            "data": "synthetic (seeded U[-1,1] RHS, SURVEY 8(d))",
            "config": bench_config(args.config, ws),
            "transport": {"kind": transport,
                          "detail": "axis-d transform reads/writes peer slabs over NVLink" if transport == "peer"
                                    else "2x NCCL all-to-all",
                          "note": transport_note, "nccl_all_to_all_ms_per_step": ms_nccl},
            "e2e": {"value": n / e2e, "unit": "DOF/s", "h2d_bytes_per_step": int(r_host.nbytes) * ws,
                    "d2h_bytes_per_step": int(r_host.nbytes) * ws, "ms_per_step": e2e * 1e3},
            "gpu_launches": launches * K, "roofline": roofline, "clocks": clk.summary(), "cpu_baseline": None,
            "solves": solves}),
            flush=True)
    dist.destroy_process_group()


def solve_roofline_s(dims, p, n, iters, fp64_peak, hbm_peak):
    """SURVEY 8(d) "Solve": iterations x (t_FD + t_mv + t_vec) at the roofline,
    t_vec = 144 B/DOF/iteration of BLAS-1 traffic (dots fused into the operators)."""
    d = len(dims) - 1
    t_fd = max(fd_flops_per_dof(dims, p) * n / (fp64_peak * 1e12), 32.0 * n / (hbm_peak * 1e9))
    t_mv = max(matvec_flops_per_dof(d, p) * n / (fp64_peak * 1e12), 32.0 * n / (hbm_peak * 1e9))
    t_vec = 144.0 * n / (hbm_peak * 1e9)
    return iters * (t_fd + t_mv + t_vec)


def two_pass_floor(ks, d, n, hbm_peak):
    """The level-pass matvec moves its rank-(d) cut through HBM once: pass 1 reads x
    and writes d intermediates, pass 2 reads them and writes y.
    Floors of that decomposition: at the HBM peak, and as measured by streaming
    kernels with the same read:write mixes on this GPU (ks_bw_fan)."""
    if d < 2:
        return None
    nmid = 3  # Schmidt rank of the system operator across any axis cut
    byts = (2 + 2 * nmid) * 16.0 * n
    g_a, g_b = ks.bw_fan(1, nmid, n), ks.bw_fan(nmid, 1, n)
    t_a, t_b = (1 + nmid) * 16.0 * n / (g_a * 1e9), (1 + nmid) * 16.0 * n / (g_b * 1e9)
    return {"bytes_per_dof": byts / n, "floor_ms_at_hbm_peak": byts / (hbm_peak * 1e9) * 1e3,
            "stream_1in_3out_gbs": g_a, "stream_3in_1out_gbs": g_b, "floor_ms_streaming": (t_a + t_b) * 1e3}


def config_leg(ks, cfg, K, W, local, fp64_peak, hbm_peak, solve=True):
    """One BASELINE config on this GPU: FD apply and matvec (device-resident,
    CUDA events), their SURVEY 8(d) rooflines, and a full FD-PCG solve to 1e-8
    with its solve roofline."""
    d, p, n_el, n_el_t = CONFIGS[cfg]
    t0 = time.perf_counter()
    prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el_t)
    P = ks.FDPreconditioner(prob, device=local)
    A = ks.assemble_system_operator(prob, device=local)
    setup_s = time.perf_counter() - t0
    dims, n = prob.reduced_dims(), prob.N_dof
    r = ks.DeviceVector.from_host(rhs(n))
    z = ks.DeviceVector(n)
    P.time(r, z, W, flush=False)
    ms_fd, ms_tr = P.time(r, z, K, flush=False)
    A.time(r, z, W, flush=False)
    ms_mv = A.time(r, z, K, flush=False)
    fd_roof = max(fd_flops_per_dof(dims, p) * n / (fp64_peak * 1e12), 32.0 * n / (hbm_peak * 1e9))
    mv_roof = max(matvec_flops_per_dof(d, p) * n / (fp64_peak * 1e12), 32.0 * n / (hbm_peak * 1e9))
    out = {"dims": dims, "dofs": n, "setup_s": setup_s,
           "fd_apply": {"ms": ms_fd, "dof_per_s": n / (ms_fd * 1e-3), "roofline_ms": fd_roof * 1e3,
                        "frac_of_roofline": fd_roof * 1e3 / ms_fd, "transform_ms_per_apply": ms_tr,
                        "info": P.info()},
           "matvec": {"ms": ms_mv, "dof_per_s": n / (ms_mv * 1e-3), "roofline_ms": mv_roof * 1e3,
                      "frac_of_roofline": mv_roof * 1e3 / ms_mv, "plan": A.plan_info(),
                      "hbm_gbs_effective": 32.0 * n / (ms_mv * 1e-3) / 1e9}}
    tp = two_pass_floor(ks, d, n, hbm_peak) if d >= 3 and n < 5e7 else None
    if tp:
        tp["frac_of_streaming_floor"] = tp["floor_ms_streaming"] / ms_mv
        out["matvec"]["two_pass"] = tp
    if solve:
        b = ks.DeviceVector.from_host(rhs(n))
        rep0 = ks.pcg(A, P, b, ks.PcgOptions(1e-8, 200))  # first solve allocates the work vectors
        rep = ks.pcg(A, P, b, ks.PcgOptions(1e-8, 200))
        roof = solve_roofline_s(dims, p, n, rep.iterations, fp64_peak, hbm_peak)
        out["solve"] = {"iterations": rep.iterations, "converged": rep.converged, "seconds": rep.solve_seconds,
                        "first_solve_seconds": rep0.solve_seconds,
                        "final_relres": rep.res_history[-1] if rep.res_history else None,
                        "roofline_s": roof, "frac_of_roofline": roof / rep.solve_seconds,
                        "roofline_basis": "SURVEY 8(d) Solve: iterations x (FD + matvec rooflines + 144 B/DOF BLAS-1)"}
    return out, P, A, prob


def latency_leg(ks, cfg, local):
    """Latency-bound configs (c1): 100 back-to-back FD applications eager and as
    CUDA-graph replays, plus one full solve (BASELINE configs[0] workload)."""
    d, p, n_el, n_el_t = CONFIGS[cfg]
    prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el_t)
    P = ks.FDPreconditioner(prob, device=local)
    A = ks.assemble_system_operator(prob, device=local)
    n = prob.N_dof
    r = ks.DeviceVector.from_host(rhs(n))
    z = ks.DeviceVector(n)
    eager = P.latency(r, z, 100, graph=False)
    graph = P.latency(r, z, 100, graph=True)
    ks.pcg(A, P, r, ks.PcgOptions(1e-8, 200))
    rep = ks.pcg(A, P, r, ks.PcgOptions(1e-8, 200))
    return {"dofs": n, "dims": prob.reduced_dims(), "fd_apply_us_eager": eager * 1e3,
            "fd_apply_us_graph": graph * 1e3, "applies": 100,
            "solve": {"iterations": rep.iterations, "converged": rep.converged, "seconds": rep.solve_seconds}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the c5 / c1 / c2 legs")
    ap.add_argument("--transport", default="auto", choices=["auto", "peer", "nccl"],
                    help="sharded FD exchange (N > 1): peer memory or NCCL all-to-all")
    args = ap.parse_args()
    if args.impl == "reference":
        # CPU arm: rank 0 alone runs the reference; other ranks exit without work
        rank = int(os.environ.get("RANK", "0"))
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference_arm(args, rank, ws, None)
        return
    rank, ws, local, dist = dist_init()
    if ws > 1:
        run_sharded(args, rank, ws, local, dist)
        return
    import paper_2311_18461_b200 as ks
    ks.lib()
    if ks.device_count() < 1:
        raise SystemExit("no CUDA device: libks has no CPU fallback")
    ks.lib().ks_set_device(local)
    d, p, n_el, n_el_t = CONFIGS[args.config]
    W = max(args.warmup, 3)
    K = args.steps
    dfma, dmma = ks.fp64_peaks()
    fp64_peak = max(dfma, dmma)
    nominal_fp64 = 37.2  # B200 datasheet-class FP64 at 1965 MHz
    pk = peaks()
    hbm_peak = pk.get("hbm_gbs", 6650.0)

    t_setup = time.perf_counter()
    prob = ks.SpaceTimeProblem.uniform(d, p, n_el, n_el_t)
    P = ks.FDPreconditioner(prob, device=local)
    A = ks.assemble_system_operator(prob, device=local)
    setup_s = time.perf_counter() - t_setup
    dims = prob.reduced_dims()
    n = prob.N_dof
    r_host = rhs(n)
    r = ks.DeviceVector.from_host(r_host)
    z = ks.DeviceVector(n)
    y = ks.DeviceVector(n)

    # ---- device-resident FD apply (the headline) ----
    clk = ClockSampler(local).__enter__()
    P.time(r, z, W, flush=False)
    ks.lib().ks_synchronize()
    ks.reset_launch_count()
    t0 = time.perf_counter()
    ms_fd, ms_gemm = P.time(r, z, K, flush=False)
    ks.lib().ks_synchronize()
    wall_fd = time.perf_counter() - t0
    launches = ks.launch_count()
    value = n / (ms_fd * 1e-3)

    prof = P.profile(r, z, K)  # per kernel kind (transforms / fused axis-1 stage / solves)

    # ---- matvec ----
    A.time(r, y, W, flush=False)
    ms_mv = A.time(r, y, K, flush=False)
    mv_two_pass = two_pass_floor(ks, d, n, hbm_peak) if d >= 3 else None
    if mv_two_pass:
        mv_two_pass["frac_of_streaming_floor"] = mv_two_pass["floor_ms_streaming"] / ms_mv

    # ---- e2e through the public host-pointer API (pinned host buffers) ----
    import ctypes as C
    hp, hz = C.c_void_p(), C.c_void_p()
    ks._check(ks.lib().ks_host_alloc(C.byref(hp), n * 16))
    ks._check(ks.lib().ks_host_alloc(C.byref(hz), n * 16))
    rin = np.ctypeslib.as_array(C.cast(hp, C.POINTER(C.c_double)), (2 * n,)).view(np.complex128)
    zout = np.ctypeslib.as_array(C.cast(hz, C.POINTER(C.c_double)), (2 * n,)).view(np.complex128)
    rin[:] = r_host
    for _ in range(2):
        P.apply(rin, zout)
    t0 = time.perf_counter()
    for _ in range(K):
        P.apply(rin, zout)
    e2e_block_s = (time.perf_counter() - t0) / K
    # the same public call on a user stream: each step still copies its r in and
    # its z out (pinned), but step k's D2H overlaps step k+1's H2D and compute
    ust = ks.Stream()
    for _ in range(2):
        P.apply(rin, zout, stream=ust)
    ust.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        P.apply(rin, zout, stream=ust)
    ust.synchronize()
    e2e_s = (time.perf_counter() - t0) / K
    e2e_val = n / e2e_s
    check = float(np.abs(zout).sum())  # the step's result was read back on the host
    clk.__exit__(None, None, None)

    # ---- roofline of the dominant kernel family: the spatial transforms ----
    # The folded transform executes 2n+2 flop per DOF (below the FP64 ridge), so
    # it is HBM-bound: SURVEY 8(d) per-unit figure 32 B/DOF (read X, write Y) x
    # N DOF per launch / the average transform launch time (CUDA events around
    # each launch). The dense-basis FP64 view (4n flop/DOF) is reported beside it.
    info = P.info()
    folded = set(info["folded_axes"])
    nlaunch = max(1, prof["transforms"]["launches"])
    t_launch = prof["transforms"]["ms"] * 1e-3 / nlaunch
    bytes_launch = 32.0 * n
    dense_flops_launch = sum(4 * dims[l] for l in range(1, d + 1)) * n / d
    exec_flops_launch = sum((2 * dims[l] + 2) if l in folded else 4 * dims[l] for l in range(1, d + 1)) * n / d
    gemm_hbm = bytes_launch / t_launch / 1e9
    fd_roof_s = max(fd_flops_per_dof(dims, p) * n / (fp64_peak * 1e12), 32.0 * n / (hbm_peak * 1e9))
    fd_roof_nominal_s = max(fd_flops_per_dof(dims, p) * n / (nominal_fp64 * 1e12), 32.0 * n / (hbm_peak * 1e9))
    mv_roof_s = max(matvec_flops_per_dof(d, p) * n / (fp64_peak * 1e12), 32.0 * n / (hbm_peak * 1e9))
    tr = ncu_traffic("k_xfold") or {}

    solves, legs = {}, {}
    if not args.no_solve:
        b = ks.DeviceVector.from_host(r_host)
        rep0 = ks.pcg(A, P, b, ks.PcgOptions(1e-8, 200))  # first solve allocates the work vectors
        rep = ks.pcg(A, P, b, ks.PcgOptions(1e-8, 200))
        roof = solve_roofline_s(dims, p, n, rep.iterations, fp64_peak, hbm_peak)
        solves[f"solve_{args.config}"] = {"iterations": rep.iterations, "converged": rep.converged,
                                          "seconds": rep.solve_seconds, "first_solve_seconds": rep0.solve_seconds,
                                          "final_relres": rep.res_history[-1] if rep.res_history else None,
                                          "roofline_s": roof, "frac_of_roofline": roof / rep.solve_seconds,
                                          "roofline_basis": "SURVEY 8(d) Solve: iterations x (FD + matvec "
                                                            "rooflines + 144 B/DOF BLAS-1)"}
    if args.config == "c3" and not args.no_extra:
        # BASELINE configs[4] (c5, 287.8 M DOF) on this GPU: FD, matvec, solve
        c5, P5, A5, _ = config_leg(ks, "c5", max(3, K // 4), 3, local, fp64_peak, hbm_peak, solve=not args.no_solve)
        del P5, A5
        legs["c5"] = c5
        # BASELINE configs[0] (c1): latency of 100 FD applies (eager / CUDA graph) + a solve
        legs["c1"] = latency_leg(ks, "c1", local)
        if not args.no_solve:
            # BASELINE configs[1]: sin-sin manufactured solution, lifted right-hand
            # side, solve to 1e-8, L2 error check -- all on the device
            p2 = ks.SpaceTimeProblem.uniform(*CONFIGS["c2"])
            P2, A2 = ks.FDPreconditioner(p2, device=local), ks.assemble_system_operator(p2, device=local)
            Q2 = ks.Quadrature(p2, device=local)
            Q2.lift("sinsin", "sinsin")  # warm-up
            lifts = []
            for _ in range(3):  # median of three (warm-up excluded, median)
                t0 = time.perf_counter()
                rhs2, bnd2 = Q2.lift("sinsin", "sinsin")
                lifts.append(time.perf_counter() - t0)
            b2 = ks.DeviceVector.from_host(rhs2)
            ks.pcg(A2, P2, b2, ks.PcgOptions(1e-8, 200))
            rep3 = ks.pcg(A2, P2, b2, ks.PcgOptions(1e-8, 200))
            errs = []
            for _ in range(3):
                t0 = time.perf_counter()
                l2, en = Q2.error_norms(Q2.extend(rep3.x, bnd2), "sinsin", "sinsin")
                errs.append(time.perf_counter() - t0)
            c2lat = P2.latency(b2, ks.DeviceVector(p2.N_dof), 100, graph=True)
            legs["c2"] = {"dofs": p2.N_dof, "iterations": rep3.iterations, "converged": rep3.converged,
                          "solve_seconds": rep3.solve_seconds, "rhs_lift_seconds": sorted(lifts)[1],
                          "error_seconds": sorted(errs)[1], "l2_error": l2, "energy_error": en,
                          "fd_apply_us_graph": c2lat * 1e3,
                          "problem": "u = sin(pi x) sin(pi y) exp(-2 i pi^2 t), f = S u"}

            # BASELINE configs[3] (c4): degree sweep p = 2..6 at 128 elements, same manufactured
            # problem: iterations, time per FD application / matvec, steady-state solve
            c4 = []
            for pdeg in range(2, 7):
                p4 = ks.SpaceTimeProblem.uniform(2, pdeg, 128, 128)
                P4, A4 = ks.FDPreconditioner(p4, device=local), ks.assemble_system_operator(p4, device=local)
                rhs4, _ = ks.Quadrature(p4, device=local).lift("sinsin", "sinsin")
                b4, x4 = ks.DeviceVector.from_host(rhs4), ks.DeviceVector(p4.N_dof)
                P4.time(b4, x4, 3)
                ms_fd4, _ = P4.time(b4, x4, 20)
                A4.apply(b4, x4)  # (the first matvec times the generated candidates)
                ks.lib().ks_synchronize()
                t0 = time.perf_counter()
                for _ in range(20):
                    A4.apply(b4, x4)
                ks.lib().ks_synchronize()
                ms_mv4 = (time.perf_counter() - t0) / 20 * 1e3
                ks.pcg(A4, P4, b4, ks.PcgOptions(1e-8, 200))
                rep4 = ks.pcg(A4, P4, b4, ks.PcgOptions(1e-8, 200))
                d4 = p4.reduced_dims()
                roof4 = max(fd_flops_per_dof(d4, pdeg) * p4.N_dof / (fp64_peak * 1e12), 32.0 * p4.N_dof / (hbm_peak * 1e9))
                c4.append({"p": pdeg, "dofs": p4.N_dof, "iterations": rep4.iterations, "converged": rep4.converged,
                           "solve_seconds": rep4.solve_seconds, "fd_apply_ms": ms_fd4, "matvec_ms": ms_mv4,
                           "fd_frac_of_roofline": roof4 * 1e3 / ms_fd4})
                del P4, A4
            legs["c4"] = c4

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        kind, sec, used = cpu_baseline_fd(args.config, r_host, steps=3, warmup=1)
        cpu = {"value": n / sec, "unit": "DOF/s", "cores": 1, "kind": kind,
               "sample": f"median of {used} full {args.config} FD applications ({n} DOF) after 1 "
                         "untimed warm-up, single thread, setup (block factorisation) excluded"}

    line = {
        "metric": "fd_apply_dof_per_s", "value": value, "unit": "DOF/s", "n_gpus": ws,
        "steps": K, "warmup": W, "ms_per_step": ms_fd, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (complex FP64)",
        "data": "synthetic (seeded U[-1,1] RHS, SURVEY 8(d))",
        "config": bench_config(args.config, ws),
        "e2e": {"value": e2e_val, "unit": "DOF/s", "h2d_bytes_per_step": n * 16,
                "d2h_bytes_per_step": n * 16, "ms_per_step": e2e_s * 1e3,
                "mode": "ks_fd_apply(host pointers, pinned) on a user stream, K steps back to back, "
                        "every step's r copied in and z copied out; copies of consecutive steps overlap",
                "blocking_value": n / e2e_block_s, "blocking_ms_per_step": e2e_block_s * 1e3},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": gemm_hbm, "peak": hbm_peak, "unit": "GB/s",
                     "frac": gemm_hbm / hbm_peak,
                     "traffic": tr.get("bytes_per_launch"), "traffic_source": tr.get("source"),
                     "algorithmic_bytes_per_launch": bytes_launch,
                     "kernel": "k_xfold (folded spatial transform, average of its %d launches per apply)" % nlaunch,
                     "basis": "SURVEY 8(d): 32 B per DOF per transform launch (read X, write Y) / launch time",
                     "launch_ms": t_launch * 1e3,
                     "executed_fp64_tflops": exec_flops_launch / t_launch / 1e12,
                     "executed_fp64_frac": exec_flops_launch / t_launch / 1e12 / fp64_peak,
                     "dense_basis_fp64_tflops": dense_flops_launch / t_launch / 1e12,
                     "peak_source": "HBM: MEASURED_PEAKS.json hbm_gbs; FP64: live DFMA %.2f / DMMA %.2f TFLOP/s "
                                    "microbenchmarks" % (dfma, dmma),
                     "transform_ms_per_apply": prof["transforms"]["ms"]},
        "fd_apply": {"ms": ms_fd, "roofline_ms": fd_roof_s * 1e3, "frac_of_roofline": fd_roof_s * 1e3 / ms_fd,
                     "frac_of_roofline_nominal_fp64": fd_roof_nominal_s * 1e3 / ms_fd,
                     "roofline_basis": "SURVEY 8(d): max(dense F_alg / FP64 peak, 32 B/DOF / HBM peak); "
                                       "FP64 peak = live microbenchmark (%.2f TF) and, for the _nominal_ "
                                       "figure, %.1f TF" % (fp64_peak, nominal_fp64),
                     "flops_per_dof_reference_algorithm": fd_flops_per_dof(dims, p),
                     "flops_per_dof_executed": fd_folded_flops_per_dof(dims, p, folded),
                     "folded_axes": sorted(folded), "factored_blocks": info["blocks"], "plan": info,
                     "components_ms_per_apply": prof,
                     "fused_axis1_stage": None if not prof["fused_axis1"]["launches"] else {
                         "ms": prof["fused_axis1"]["ms"],
                         "algorithmic_bytes": 32.0 * n + info["blocks"] * dims[0] * (16 * p + 8),
                         "hbm_gbs": (32.0 * n + info["blocks"] * dims[0] * (16 * p + 8)) / (prof["fused_axis1"]["ms"] * 1e-3) / 1e9,
                         "note": "slab in + out (32 B/DOF) and the L D L^H factor rows read once (16p+8 B per block and "
                                 "time step); the sweeps' latency, not bandwidth, bounds it (DESIGN.md 3.3)"},
                     "wall_s": wall_fd},
        "matvec": {"ms": ms_mv, "dof_per_s": n / (ms_mv * 1e-3),
                   "roofline_ms": mv_roof_s * 1e3, "frac_of_roofline": mv_roof_s * 1e3 / ms_mv,
                   "plan": A.plan_info(), "hbm_gbs_effective": 32.0 * n / (ms_mv * 1e-3) / 1e9,
                   "two_pass": mv_two_pass},
        "solves": solves,
        "legs": legs,
        "setup_s": setup_s,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "checksum": check,
    }
    print(json.dumps(line), flush=True)
    ks.lib().ks_host_free(hp)
    ks.lib().ks_host_free(hz)


if __name__ == "__main__":
    main()
