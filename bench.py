#!/usr/bin/env python
"""Benchmark of the GPSS iteration loop (BASELINE.json metric: projected-gradient
iterations/s and achieved HBM GB/s of K streamed vs peak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl b200|reference]

A step is one gpss_solve of the config with K resident in HBM.  The default workload is C4
(BASELINE.json configs[3]: 32768x262144 Gaussian, 68.7 GB, 200 iterations, x0 = 0) at every
N, the config the north star's multi-GPU target names; it fits one 180 GB B200, so the N=1
line of the scaling run is the same workload (--config C1/C2/C3/C5 select the others).  K
is larger than L2, so no flush is needed between steps.  With N > 1 the problem is
column-sharded over the N GPUs (strong scaling); `--gpus N` launches the N ranks itself
(torch.distributed.run) when it is not already running under a launcher.
`value` = iterations / device time (CUDA events on the solver stream, max over ranks);
`e2e` = the same metric through the C-ABI call l1g_gpss_solve with host y and x buffers
(copies inside the timed region).  Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "projected-gradient iterations/s"
UNIT = "iterations/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def sigma_fixture(name):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        mx = float(rows[0][2])
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows)}


def spawn_if_needed(args):
    """`--gpus N` with no launcher around us: re-run this command under torch.distributed.run
    with N ranks (127.0.0.1 rendezvous) and exit with its code.  Under a launcher the world
    size must equal N."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            sys.exit(2)
        return
    if args.gpus <= 1:
        return
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


def max_over_ranks(pg, v):
    if pg is None:
        return v
    import torch
    dev = "cuda" if pg.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


# ------------------------------------------------------------------ CPU baseline (oracle)
def host_ram_gb():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) / 2**20
    except Exception:
        pass
    return 0.0


def omp_threads(n):
    """Thread count of the OpenMP runtime the oracle and oracle/_ref share (libgomp)."""
    import ctypes as C
    try:
        C.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


class CpuRef:
    """The reference's CPU path on this host.  kind "reference": the reference's own
    gpss.cpp/prox.cpp/linear_operator.cpp (oracle/_ref/libref_fast.so: Eigen stand-in with
    OpenMP GEMVs over outputs and sequential sums); it keeps its own column-major copy of K.
    kind "port": the oracle's restatement in LITERAL mode on the row-major K in place -- the
    same arithmetic (bit-identical records and iterates on every config of
    profiles/r02_divergence.json), used when the host cannot hold the second copy (C4)."""

    def __init__(self, K, kind):
        from oracle import ref as R
        self.K, self.kind = K, kind
        self.op = R.RefOperator(K, "fast") if kind == "reference" else None

    def solve(self, y, rho, iters, threads=None):
        from oracle import oracle as O
        omp_threads(threads or (os.cpu_count() or 1))
        stop = O.StopRule(iters, 0, 0, 0.0)
        t0 = time.perf_counter()
        if self.op is not None:
            _, res, _ = self.op.gpss_solve(y, rho, O.GpConfig(), stop, trace=False)
        else:
            with O.mode(O.LITERAL):
                _, res, _, _ = O.gpss_solve(self.K, y, rho, O.GpConfig(), stop, trace=False)
        dt = time.perf_counter() - t0
        omp_threads(os.cpu_count() or 1)
        return dt, res["iterations"]


def cpu_ref_for(K):
    """The reference's own sources when the host can hold their column-major copy of K next
    to ours, else the literal-mode port on K in place."""
    from oracle import ref as R
    gb = K.nbytes / 2**30
    if R.available("fast") and host_ram_gb() > 1.2 * gb + 4:
        return CpuRef(K, "reference")
    return CpuRef(K, "port")


def host_fits(cfgname):
    """None when the host can hold the config's K, else the reason."""
    from tests import problems as PB
    if cfgname == "C5":
        return None
    spec = getattr(PB, cfgname)
    need = spec.n * spec.p * 8 / 2**30 * 1.1 + 4
    have = host_ram_gb()
    if have < need:
        return (f"host RAM: {cfgname} needs ~{need:.0f} GiB for K on the host, "
                f"{have:.0f} GiB available")
    return None


def cpu_sample(cref, y, rho, target_s, cap, threads=None):
    """A bounded sample: enough iterations for ~target_s of CPU work (>= 1)."""
    dt1, it1 = cref.solve(y, rho, 1, threads)
    per = max(1, min(cap, int(target_s * max(it1, 1) / max(dt1, 1e-4))))
    if per == 1:
        return dt1, it1, 1
    dt, itn = cref.solve(y, rho, per, threads)
    return dt, itn, per


def cpu_leg(K, y, rho, label, per_unit=1):
    """cpu_baseline of the b200 arm: the reference CPU path on a bounded sample of the same
    workload, with all host threads and (the reference's own setting) with one thread."""
    cref = cpu_ref_for(K)
    cores = os.cpu_count() or 1
    dt, itn, _ = cpu_sample(cref, y, rho, 12.0, 400)
    dt1, itn1, _ = cpu_sample(cref, y, rho, 8.0, 400, threads=1)
    src = ("reference sources via oracle/_ref/libref_fast.so, OpenMP GEMVs"
           if cref.kind == "reference" else
           "oracle LITERAL mode (bit-identical to the reference sources), OpenMP GEMVs")
    return {"value": itn / dt / per_unit, "unit": UNIT, "cores": cores, "kind": cref.kind,
            "sample": f"{itn} GPSS iterations (incl. gp_init) of {label} from x0=0, {src}, "
                      f"{cores} threads" + (f", scaled to lockstep iterations (/{per_unit})"
                                            if per_unit > 1 else ""),
            "single_thread": {"value": itn1 / dt1 / per_unit, "cores": 1,
                              "sample": f"{itn1} iterations, 1 thread: the reference's own "
                                        "build has no OpenMP and Eigen's GEMV is "
                                        "single-threaded"}}


def host_problem(spec_name):
    """The config's problem built on the host with the oracle generators and canonical
    reductions (bit-identical to the device build: tests/test_gpu_fullsize_parity.py)."""
    import copy

    from oracle import oracle as O
    from tests import problems as PB
    spec = copy.copy(getattr(PB, spec_name))
    if spec.kind == "gaussian":
        spec.sigma_hat = sigma_fixture(spec_name)
        if spec.sigma_hat is None:  # short power iteration as a stand-in scale (timing only)
            spec.power_iters = 8
    P = O.build_problem(spec)
    return P["K"], P["y"], float(P["rho"])


def host_batch_problem0():
    """C5 (BASELINE configs[4]) problem 0 on the host with the oracle generators (the same
    streams harness.build_batch_problem uses on the device)."""
    from oracle import oracle as O
    from paper_0902_4424_b200 import harness as H
    c = H.C5
    n, p, seed = c["n"], c["p"], c["seed"]
    K = O.gaussian_matrix(seed, n, p)
    sigma = sigma_fixture("C5")
    if sigma is None:
        sigma, _ = O.spectral_norm(K, 8, 1e-8)
    O.lib().orc_scale(K, K.size, 0.9 / sigma)
    sj = 1000 * seed
    spec = O.ProblemSpec("gaussian", n, p, c["nnz"], sj, "normal", c["noise"], "abs")
    x = np.zeros(p)
    x[O.sample_support(sj, 1, p, c["nnz"])] = O.x_true_values(spec, c["nnz"])
    y = O.apply(K, x) + c["noise"] * O.fill_normal(sj, 2, 0, n)
    return K, y, 0.2 * O.l1norm(x), c["batch"]


def run_reference(args, world, rank, pg):
    """--impl reference: the reference CPU path on this box's host cores (all threads)."""
    if rank != 0:
        return
    cfgname = args.config
    scale = 1
    why = host_fits(cfgname)
    if why is not None:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return
    t_setup = time.perf_counter()
    if cfgname == "C5":  # problems are solved one by one there: lockstep unit = B problems
        K, y, rho, scale = host_batch_problem0()
    else:
        K, y, rho = host_problem(cfgname)
    cref = cpu_ref_for(K)
    setup_s = time.perf_counter() - t_setup
    n, p = K.shape
    cores = os.cpu_count() or 1
    # bounded sample per step, sized so all warmup + timed steps take ~2-3 minutes
    dt1, it1 = cref.solve(y, rho, 1)
    budget = 150.0 / max(1, args.steps + args.warmup)
    per_step = max(1, min(args.ref_iters or 1000, int(budget * max(it1, 1) / max(dt1, 1e-3))))
    for _ in range(args.warmup):
        cref.solve(y, rho, per_step)
    times, total_it = [], 0
    for _ in range(args.steps):
        dt, itn = cref.solve(y, rho, per_step)
        times.append(dt)
        total_it += itn
    total_t = sum(times)
    v = total_it / total_t / scale
    src = ("reference gpss.cpp/prox.cpp/linear_operator.cpp via oracle/_ref/libref_fast.so "
           "(Eigen stand-in: OpenMP GEMVs over outputs, sequential sums)"
           if cref.kind == "reference" else
           "oracle restatement in LITERAL mode (the reference's arithmetic, bit-identical to "
           "oracle/_ref/libref_fast.so; K row-major in place)")
    sample = (f"{per_step} GPSS iterations per step of {cfgname} ({n}x{p}) from x0=0, "
              + (f"problem 0 of {scale} solved alone, scaled to lockstep iterations (/{scale}), "
                 if scale > 1 else "") + src + f", {cores} threads")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox Gaussian, oracle generator on the host)",
            "config": {"workload": cfgname, "n": n, "p": p, "iterations_per_step": per_step,
                       "setup_s": round(setup_s, 1)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": cref.kind,
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gbs_K": v * 2 * n * p * 8 / 1e9}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ C5: batched RHS
def fp64_peak():
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            return float(json.load(f)["dmma_m8n8k4_tflops"]), "measured (tools/fp64_peak.cu)"
    except Exception:
        return 37.0, "fallback"


def run_batch(args, world, rank, local, pg):
    """BASELINE configs[4]: 128 problems on one 4096x16384 K, solved in lockstep; the
    products run on the FP64 tensor cores.  A step is one batched gpss_solve (all problems
    to their stop rule, at most 300 lockstep iterations)."""
    import ctypes as C

    import paper_0902_4424_b200 as l1
    from paper_0902_4424_b200 import _lib as L
    from paper_0902_4424_b200 import harness as H

    import torch
    torch.cuda.set_device(local)
    c = dict(H.C5)
    B, n, p = c["batch"], c["n"], c["p"]
    iters = args.iters or H.ITERATIONS["C5"]
    t_setup = time.perf_counter()
    P = H.build_batch_problem(**c, sigma_hat=sigma_fixture("C5"))
    setup_s = time.perf_counter() - t_setup
    lib = L.load()
    cfg = l1.GpConfig()._c()
    stop = l1.StopRule(max_iterations=iters, stationarity_tol=0.0)._c()
    Y = np.ascontiguousarray(P["Y"])
    rho = np.ascontiguousarray(P["rho"])
    h = C.c_void_p()
    L.check(lib.l1g_batch_create(P["op"].h, B, L.ptr(Y), L.ptr(rho), C.byref(cfg), C.byref(h)))
    sp = C.c_void_p()
    lib.l1g_batch_stream(h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    res = (L.ResultC * B)()

    def solve_once():
        L.check(lib.l1g_batch_init(h, None), "batch_init")
        L.check(lib.l1g_batch_run(h, C.byref(stop), res), "batch_run")
        its = [res[i].iterations for i in range(B)]
        return max(its), sum(its)

    for _ in range(args.warmup):
        solve_once()
    tl = C.c_int64()
    lib.l1g_batch_launches(h, C.byref(tl), 1)
    barrier(pg)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lock_its = prob_its = 0
    with clocks:
        e0.record(stream)
        for _ in range(args.steps):
            a, b = solve_once()
            lock_its += a
            prob_its += b
        e1.record(stream)
        e1.synchronize()
    dev_ms = max_over_ranks(pg, e0.elapsed_time(e1))
    lib.l1g_batch_launches(h, C.byref(tl), 1)
    value = world * lock_its / (dev_ms / 1e3)
    tf, ta = C.c_double(), C.c_double()
    L.check(lib.l1g_batch_time_products(h, 10, C.byref(tf), C.byref(ta)))
    X_dev = np.empty((B, p))
    L.check(lib.l1g_batch_get_x(h, L.ptr(X_dev)))
    lib.l1g_batch_destroy(h)

    # end to end: l1g_gpss_solve_batched with host Y / rho in and X / results out, the host
    # buffers pinned (page-locked) as the contract asks
    Yh = torch.empty((B, n), dtype=torch.float64, pin_memory=True).numpy()
    Yh[:] = Y
    X = torch.empty((B, p), dtype=torch.float64, pin_memory=True).numpy()
    res2 = (L.ResultC * B)()

    def e2e_once():
        L.check(lib.l1g_gpss_solve_batched(P["op"].h, B, L.ptr(Yh), L.ptr(rho), C.byref(cfg),
                                           C.byref(stop), L.ptr(X), res2), "solve_batched")
        return max(res2[i].iterations for i in range(B))

    e2e_once()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_its = sum(e2e_once() for _ in range(max(1, args.steps // 2)))
    e2e_s = max_over_ranks(pg, time.perf_counter() - t0)

    peak, peak_src = fp64_peak()
    flop = 2.0 * n * p * B  # one product
    dom = "adj" if ta.value >= tf.value else "fwd"
    ms = {"fwd": tf.value, "adj": ta.value}[dom]
    achieved = flop / (ms / 1e3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get({"adj": "C5_badj", "fwd": "C5_bfwd"}[dom])
    except Exception:
        pass
    roofline = {"bound": "tensor", "kernel": {"adj": "badj_kernel (K^T R', DMMA)",
                                              "fwd": "bfwd_kernel (K D, DMMA)"}[dom],
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": peak_src, "traffic": traffic,
                "traffic_unit": "bytes per launch (K 512 MiB + vectors + split partials)",
                "algorithmic_flops_per_launch": flop,
                "avg_launch_ms": {"bfwd": round(tf.value, 4), "badj": round(ta.value, 4)},
                "iteration_TFLOPs_4npB": 2 * flop * lock_its / (dev_ms / 1e3) / 1e12}
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            K = P["op"].matrix()
            cpu = cpu_leg(K, Y[0], float(rho[0]), f"problem 0 of C5 solved alone", per_unit=B)
            del K
        except Exception as ex:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {ex}"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64",
                "data": "synthetic (seeded Philox Gaussian K scaled to ||K||_2=0.9 on device, "
                        "128 seeded x_true; BASELINE.json configs[4])",
                "config": {"workload": f"C5: batched {B} problems on gaussian {n}x{p}, nnz 150 "
                                       f"each, rho_j = (0.2..1.0)||x_true_j||_1, up to {iters} "
                                       "lockstep iterations, x0=0, stationarity_tol=0",
                           "n": n, "p": p, "batch": B,
                           "lockstep_iterations_per_step": lock_its / args.steps,
                           "problem_iterations_per_s": world * prob_its / (dev_ms / 1e3),
                           "l2": "inputs larger than L2 (K = 0.5 GiB, partials 67 MB)",
                           "products": "on the live problems only: stopped problems are "
                                       "compacted out of the DMMA products (problem blocks, "
                                       "32-problem warp groups and 8-problem tiles without a live "
                                       "problem are skipped; same bits per problem); the "
                                       "roofline launches below are full-width (all problems)",
                           "mean_live_problems": prob_its / max(lock_its, 1),
                           "parallelism": "replicas" if world > 1 else "single",
                           "setup_s": round(setup_s, 3)},
                "e2e": {"value": world * e2e_its / e2e_s, "unit": UNIT,
                        "h2d_bytes_per_step": Y.nbytes + rho.nbytes,
                        "d2h_bytes_per_step": X.nbytes + B * C.sizeof(L.ResultC),
                        "x_matches_device_run": bool(np.array_equal(X, X_dev))},
                "gpu_launches": int(tl.value),
                "roofline": roofline,
                "cpu_baseline": cpu,
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def run_b200(args, world, rank, local, pg):
    import ctypes as C

    import paper_0902_4424_b200 as l1
    from paper_0902_4424_b200 import _lib as L
    from paper_0902_4424_b200 import harness as H

    import torch
    torch.cuda.set_device(local)
    ctx = l1.Context(local)
    spec = H.CONFIGS[args.config]
    iters = args.iters or H.ITERATIONS[args.config]
    fix = sigma_fixture(args.config)
    t_setup = time.perf_counter()
    if fix is not None and not args.recompute_sigma:
        spec.sigma_hat = fix
    P = H.build_problem(spec, ctx)
    op, y, rho = P["op"], P["y"], P["rho"]
    n, p = spec.n, spec.p
    lib = L.load()
    cfg = l1.GpConfig()._c()
    stop = l1.StopRule(max_iterations=iters, stationarity_tol=0.0)._c()
    comm = None
    h = C.c_void_p()
    sharded = world > 1 or args.force_sharded
    if sharded:
        # column sharding over the ranks: this rank keeps only its block of
        # columns; y and rho come from the full problem built above (identical on all ranks)
        from paper_0902_4424_b200 import shard as S
        if spec.sigma_hat is None:
            spec.sigma_hat = P["sigma_hat"]
        sh = S.shard_plan(p, world)[rank]
        op.close()
        op, _, _ = H.build_operator(spec, ctx, col_offset=sh.col0, p_local=sh.p_local)
        if pg is not None:
            uid = S.exchange_id(pg, rank)
        else:
            buf = (C.c_uint8 * 128)()
            L.check(lib.l1g_comm_unique_id(C.cast(buf, C.c_void_p)), "comm_unique_id")
            uid = bytes(buf)
        comm = S.Comm(ctx, rank, world, uid)
        h = S.create_sharded_solver(op, comm, y, rho, l1.GpConfig())
    else:
        # ---- device-resident solver (inputs already in HBM)
        L.check(lib.l1g_solver_create(op.h, L.ptr(np.ascontiguousarray(y)), rho, C.byref(cfg),
                                      C.byref(h)), "solver_create")
    setup_s = time.perf_counter() - t_setup
    sp = C.c_void_p()
    lib.l1g_solver_stream(h, C.byref(sp))
    stream = torch.cuda.ExternalStream(sp.value)
    res = L.ResultC()

    def solve_once():
        L.check(lib.l1g_solver_init(h, None), "init")
        L.check(lib.l1g_solver_run(h, C.byref(stop), C.byref(res), None, 0), "run")
        return res.iterations

    for _ in range(args.warmup):
        solve_once()
    lib.l1g_solver_timing(h, None, None, None, None, None, 1)
    barrier(pg)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    done_iters = 0
    with clocks:
        e0.record(stream)
        for _ in range(args.steps):
            done_iters += solve_once()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
    barrier(pg)
    dev_ms = e0.elapsed_time(e1)
    dev_ms = max_over_ranks(pg, dev_ms)
    tp, tf, ta = C.c_double(), C.c_double(), C.c_double()
    ti, tl = C.c_int64(), C.c_int64()
    lib.l1g_solver_timing(h, None, None, None, None, C.byref(tl), 1)
    value = done_iters / (dev_ms / 1e3)  # iterations/s of the one (sharded) problem
    reason = L.REASONS[res.reason]
    # per-kernel breakdown: a separate solve with event nodes between the kernels (they
    # serialise the programmatic launches, so this pass is not the timed one)
    L.check(lib.l1g_solver_set_timing(h, 1))
    solve_once()
    lib.l1g_solver_timing(h, C.byref(tp), C.byref(tf), C.byref(ta), C.byref(ti), None, 1)
    L.check(lib.l1g_solver_set_timing(h, 0))
    nccl = None
    if sharded:  # the two allgathers of an iteration, timed alone on the solver stream
        xk, xg = C.c_double(), C.c_double()
        L.check(lib.l1g_solver_time_exchange(h, 20, C.byref(xk), C.byref(xg)), "time_exchange")
        nccl = {"allgather_Kd_ms": round(max_over_ranks(pg, xk.value), 5),
                "allgather_xg_packet_ms": round(max_over_ranks(pg, xg.value), 5),
                "share_of_iteration": round((xk.value + xg.value) /
                                            (dev_ms / max(done_iters, 1)), 4)}
    prof = (C.c_double * 32)()
    lib.l1g_solver_proj_profile(h, prof)
    sp_cols = prof[18] / prof[19] if prof[19] > 0 else None

    # ---- end to end through the C-ABI with host buffers (pinned)
    yp, xp = C.c_void_p(), C.c_void_p()
    L.check(lib.l1g_host_alloc(n * 8, C.byref(yp)))
    L.check(lib.l1g_host_alloc(p * 8, C.byref(xp)))
    np.ctypeslib.as_array((C.c_double * n).from_address(yp.value))[:] = y
    res2 = L.ResultC()

    def e2e_once():
        if sharded:  # the sharded solver's public calls, host y in, host x out
            L.check(lib.l1g_solver_set_y(h, yp), "set_y")
            L.check(lib.l1g_solver_init(h, None), "init")
            L.check(lib.l1g_solver_run(h, C.byref(stop), C.byref(res2), None, 0), "run")
            L.check(lib.l1g_solver_get(h, xp, None, None, None, None, None, None), "get")
            return res2.iterations
        L.check(lib.l1g_gpss_solve(op.h, yp, rho, C.byref(cfg), C.byref(stop), None, xp,
                                   C.byref(res2), None, 0), "gpss_solve")
        return res2.iterations

    for _ in range(max(1, args.warmup)):
        e2e_once()
    barrier(pg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_iters = 0
    for _ in range(args.steps):
        e2e_iters += e2e_once()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(pg, time.perf_counter() - t0)
    e2e_value = e2e_iters / e2e_s
    x_e2e = np.ctypeslib.as_array((C.c_double * p).from_address(xp.value)).copy()
    x_dev = np.empty(p)
    L.check(lib.l1g_solver_get(h, L.ptr(x_dev), None, None, None, None, None, None))
    lib.l1g_host_free(yp)
    lib.l1g_host_free(xp)

    # ---- roofline of the dominant kernel (per-launch CUDA events inside the timed loop)
    hbm, peak_src = peaks()
    k_bytes = n * p * 8.0 / world  # this rank's columns
    it = max(ti.value, 1)
    avg = {"proj": tp.value / it, "fwd": tf.value / it, "adj": ta.value / it}
    dom = "adj" if avg["adj"] >= avg["fwd"] else "fwd"
    achieved = k_bytes / (avg[dom] / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.config}_{dom}")
    except Exception:
        pass
    small = C.c_int(0)
    if hasattr(lib, "l1g_solver_small_path"):
        lib.l1g_solver_small_path(h, C.byref(small))
    roofline = {"bound": "hbm", "kernel": {"adj": "adj_kernel (2 K^T r)",
                                           "fwd": "fwd_sparse_kernel (K d)"}[dom],
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_source": peak_src, "traffic": traffic,
                "algorithmic_bytes_per_launch": k_bytes,
                "avg_launch_ms": {k: round(v, 5) for k, v in avg.items()},
                "fwd_sparse": None if sp_cols is None else {
                    "support_columns_per_call": round(sp_cols, 1),
                    "K_bytes_per_call": sp_cols * n * 8.0,
                    "GBps_incl_finish": sp_cols * n * 8.0 / (avg["fwd"] / 1e3) / 1e9},
                "share_of_iteration": {k: round(v / sum(avg.values()), 4)
                                       for k, v in avg.items()},
                # K bytes the iteration actually reads (adjoint: all of K; forward: the
                # support columns of d), per second of the timed solves
                "iteration_GBps_K_read": None if sp_cols is None else
                (k_bytes + sp_cols * n * 8.0) * done_iters / (dev_ms / 1e3) / 1e9,
                "iteration_frac_K_read": None if sp_cols is None else
                (k_bytes + sp_cols * n * 8.0) * done_iters / (dev_ms / 1e3) / 1e9 / hbm,
                "nominal_iteration_GBps_2npx8": 2 * k_bytes * done_iters / (dev_ms / 1e3) / 1e9}
    if small.value:  # K (L2-resident) staged once per iteration into one cluster's shared memory
        sm_ms = avg["fwd"] + avg["adj"]
        roofline.update({
            "bound": "latency",
            "kernel": "small_iter_kernel (K d, line search, K^T r', step; K tiles in shared memory)",
            "achieved": k_bytes / (sm_ms / 1e3) / 1e9, "frac": k_bytes / (sm_ms / 1e3) / 1e9 / hbm,
            "note": "K fits L2 and one cluster's shared memory: the iteration is two kernels "
                    "(projection, step) of dependent on-chip reductions, so HBM bandwidth does "
                    "not bound it; achieved = K bytes staged per step kernel / its time",
            "fwd_sparse": None, "iteration_GBps_K_read": None, "iteration_frac_K_read": None})

    # ---- CPU baseline on rank 0 at N=1 (bounded sample of the same workload)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        why = host_fits(args.config)
        if why is not None:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"skipped: {why}"}
        else:
            try:
                Kh, yh, rhoh = host_problem(args.config)  # same bits as the device build
                cpu = cpu_leg(Kh, yh, rhoh, args.config)
                del Kh
            except Exception as ex:  # reported, never fatal
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                       "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded Philox streams, generated on device; BASELINE.json "
                        f"configs[{int(args.config[1]) - 1}])",
                "config": {"workload": f"{args.config}: {spec.kind} {n}x{p}, nnz {spec.nnz}, "
                                       f"{iters} iterations, x0=0, stationarity_tol=0",
                           "n": n, "p": p, "iterations_per_step": done_iters / args.steps,
                           "stop_reason": reason, "rho": rho, "sigma_hat": P["sigma_hat"],
                           "l2": ("inputs larger than L2 (K = %.2f GiB)" % (k_bytes / 2**30))
                                 if k_bytes > 126e6 else
                                 "K = %.1f MiB is L2-resident (a latency-bound config)" % (k_bytes / 2**20),
                           "parallelism": (f"column-sharded over {world} GPUs (rank-owned x, g "
                                           "slices; NCCL allgathers of the K d shard values "
                                           "and of the [x | g | dots] packets)")
                           if sharded else "single",
                           "setup_s": round(setup_s, 3)},
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * 8,
                        "d2h_bytes_per_step": p * 8 + C.sizeof(L.ResultC),
                        "x_matches_device_run": bool(np.array_equal(x_e2e, x_dev))},
                "gpu_launches": int(tl.value),
                "roofline": roofline,
                "cpu_baseline": cpu,
                "clocks": clocks.summary()}
        if nccl is not None:
            line["nccl"] = nccl
        print(json.dumps(line), flush=True)
    lib.l1g_solver_destroy(h)
    if comm is not None:
        comm.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--recompute-sigma", action="store_true")
    ap.add_argument("--ref-iters", type=int, default=0)
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the NCCL-sharded solver path even on one GPU (a 1-rank communicator)")
    args = ap.parse_args()
    spawn_if_needed(args)
    world, rank, local, pg = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank, pg)
    elif args.config == "C5":
        run_batch(args, world, rank, local, pg)
    else:
        run_b200(args, world, rank, local, pg)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
