"""Short solve for profiling (ncu launch lists / --set full captures).

  python tools/prof_solve.py --config C2 --iters 20 [--solves 1]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_0902_4424_b200 as l1  # noqa: E402
from paper_0902_4424_b200 import _lib as L  # noqa: E402
from paper_0902_4424_b200 import harness as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--solves", type=int, default=1)
    ap.add_argument("--profile", action="store_true", help="print projection phase profile")
    ap.add_argument("--timing", action="store_true", help="per-kernel CUDA-event timing")
    ap.add_argument("--trace", action="store_true", help="print per-iteration support sizes")
    a = ap.parse_args()
    spec = H.CONFIGS[a.config]
    fx = os.path.join(ROOT, "tests", "golden", "sigma_hat.json")
    if os.path.exists(fx):
        spec.sigma_hat = json.load(open(fx)).get(a.config)
    P = H.build_problem(spec)
    lib = L.load()
    cfg = l1.GpConfig()._c()
    stop = l1.StopRule(max_iterations=a.iters, stationarity_tol=0.0)._c()
    h = C.c_void_p()
    L.check(lib.l1g_solver_create(P["op"].h, L.ptr(np.ascontiguousarray(P["y"])), P["rho"],
                                  C.byref(cfg), C.byref(h)))
    res = L.ResultC()
    if a.timing:
        L.check(lib.l1g_solver_set_timing(h, 1))
    for s in range(a.solves):
        t = time.perf_counter()
        L.check(lib.l1g_solver_init(h, None))
        cap = a.iters if a.trace else 0
        recs = (L.IterRecordC * max(cap, 1))()
        L.check(lib.l1g_solver_run(h, C.byref(stop), C.byref(res),
                                   C.addressof(recs) if cap else None, cap))
        dt = time.perf_counter() - t
        print(f"solve {s}: {res.iterations} iterations ({L.REASONS[res.reason]}) in {dt*1e3:.2f} ms"
              f" = {res.iterations / dt:.1f} it/s, f={res.objective:.6e}", flush=True)
    if a.trace:
        sup = [recs[i].support for i in range(min(res.iterations, a.iters))]
        print("support per iteration:", sup)
        print("alpha per iteration:", [f"{recs[i].alpha:.3g}" for i in range(min(res.iterations, a.iters))])
    if a.timing:
        tp, tf, ta, ti, tl = (C.c_double(), C.c_double(), C.c_double(), C.c_int64(),
                              C.c_int64())
        lib.l1g_solver_timing(h, C.byref(tp), C.byref(tf), C.byref(ta), C.byref(ti),
                              C.byref(tl), 0)
        it = max(ti.value, 1)
        kb = spec.n * spec.p * 8
        print(f"per iteration ms: proj {tp.value/it:.4f} fwd {tf.value/it:.4f} "
              f"adj {ta.value/it:.4f}  GB/s fwd {kb/(tf.value/it)/1e6:.0f} "
              f"adj {kb/(ta.value/it)/1e6:.0f}  ({it} iterations, {tl.value} launches)")
    if a.profile and hasattr(lib, "l1g_solver_proj_profile"):
        out = (C.c_double * 24)()
        lib.l1g_solver_proj_profile(h, out)
        print("proj profile:", [round(v, 3) for v in out])
        if out[19] > 0:
            cols = out[18] / out[19]
            print(f"sparse forward: {cols:.1f} support columns per call "
                  f"({cols / spec.p:.3%} of p), {cols * spec.n * 8 / 1e6:.1f} MB of K per call")
    if hasattr(lib, "l1g_debug_prefix_trace"):  # L1G_PROJ_TRACE builds: the last prefix call
        tr, stp = (C.c_longlong * 192)(), (C.c_longlong * 520)()
        lib.l1g_debug_prefix_trace(tr, stp)
        print("prefix head: seq %d test %d sync %d" % (stp[513] - stp[512], stp[514] - stp[513],
                                                      stp[515] - stp[514]))
        for e in range(64):
            if tr[3 * e] == 0:
                break
            st = [stp[e * 8 + k] - tr[3 * e] if stp[e * 8 + k] else -1 for k in range(6)]
            print(f"  epoch {e}: t={tr[3 * e] - tr[0]} i0={tr[3 * e + 1]} window={tr[3 * e + 2]}"
                  f" stamps={st}")
    lib.l1g_solver_destroy(h)


if __name__ == "__main__":
    main()
