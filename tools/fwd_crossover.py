"""Density crossover of the iteration's forward product: support gather (fwd_sparse_kernel)
versus the dense TMA stream (fwd_kernel), timed in situ on C2-shaped problems whose radius
rho = f * ||x_true||_1 sets how dense the directions d are.

  python tools/fwd_crossover.py [--config C2] [--iters 30] > profiles/r02_fwd_crossover.txt

Per rho factor: the mean fraction of nonzero columns in d (sparse run telemetry), and the
event-timed forward phase (kernel + finish) per iteration in mode 2 (sparse only), mode 0
(dense only) and mode 1 (sparse with the device-side switch at L1G_FWD_DENSE_FRAC)."""
import argparse
import ctypes as C
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_0902_4424_b200 as l1  # noqa: E402
from paper_0902_4424_b200 import _lib as L  # noqa: E402
from paper_0902_4424_b200 import harness as H  # noqa: E402
from paper_0902_4424_b200 import shard as S  # noqa: E402


def timed(lib, P, mode, iters):
    h = C.c_void_p()
    cfg = l1.GpConfig()._c()
    L.check(lib.l1g_solver_create(P["op"].h, L.ptr(np.ascontiguousarray(P["y"])), P["rho"],
                                  C.byref(cfg), C.byref(h)))
    try:
        L.check(lib.l1g_solver_set_forward(h, mode))
        L.check(lib.l1g_solver_set_timing(h, 1))
        S.solve(h, l1.StopRule(max_iterations=iters, stationarity_tol=0.0))  # warm
        res, _ = S.solve(h, l1.StopRule(max_iterations=iters, stationarity_tol=0.0))
        tp, tf, ta, ti, tl = (C.c_double(), C.c_double(), C.c_double(), C.c_int64(),
                              C.c_int64())
        lib.l1g_solver_timing(h, C.byref(tp), C.byref(tf), C.byref(ta), C.byref(ti),
                              C.byref(tl), 0)
        prof = (C.c_double * 32)()
        L.check(lib.l1g_solver_proj_profile(h, prof))
        it = max(ti.value, 1)
        return tf.value / it, prof[18] / max(prof[19], 1.0), prof[23], res.iterations
    finally:
        lib.l1g_solver_destroy(h)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--factors", default="1,1.5,2,3,4,6,10")
    a = ap.parse_args()
    sig = json.load(open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")))
    base = H.CONFIGS[a.config]
    lib = L.load()
    kbytes = base.n * base.p * 8
    print(f"# {a.config} {base.n}x{base.p}: forward phase per iteration (fwd kernel + finish, "
          f"CUDA events, mean over {a.iters} iterations after a warm run)")
    print("rho_factor  d_density  sparse_ms  dense_ms  switch_ms  switch_dense_calls  "
          "sparse_GBps_on_support  dense_GBps")
    for f in [float(v) for v in a.factors.split(",")]:
        spec = dataclasses.replace(base, rho_factor=f, sigma_hat=sig.get(a.config))
        P = H.build_problem(spec)
        ts, cols, _, _ = timed(lib, P, 2, a.iters)
        td, _, _, _ = timed(lib, P, 0, a.iters)
        tw, _, nd, _ = timed(lib, P, 1, a.iters)
        dens = cols / base.p
        print(f"{f:10.2f}  {dens:9.3f}  {ts:9.4f}  {td:8.4f}  {tw:9.4f}  {int(nd):18d}  "
              f"{dens * kbytes / ts / 1e6:22.0f}  {kbytes / td / 1e6:10.0f}", flush=True)


if __name__ == "__main__":
    main()
