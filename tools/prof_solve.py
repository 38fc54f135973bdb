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

if "--timeline" in sys.argv:  # the L1G_TIMELINE build (paper_0902_4424_b200.build.build_variant)
    os.environ["L1G_LIB_PATH"] = os.path.join(ROOT, "paper_0902_4424_b200", "libl1g_tl.so")

import numpy as np  # noqa: E402

import paper_0902_4424_b200 as l1  # noqa: E402
from paper_0902_4424_b200 import _lib as L  # noqa: E402
from paper_0902_4424_b200 import harness as H  # noqa: E402


def timeline(lib, iters):
    """Per kernel: mean in-graph phase (start after griddepcontrol.wait to the next kernel's),
    and how early its first CTA entered before the wait released."""
    g, pj = (C.c_ulonglong * 4096)(), (C.c_ulonglong * 4096)()
    lib.l1g_debug_timeline_gemv(g, 0)
    lib.l1g_debug_timeline_proj(pj, 0)
    t = np.minimum(np.frombuffer(g, dtype=np.uint64), np.frombuffer(pj, dtype=np.uint64))
    t = t.reshape(256, 16).astype(np.float64)
    names = ["proj", "fwd_sparse", "fwd_finish", "adj", "adj_finish"]
    ks = [k for k in range(5, min(iters, 256) - 1) if np.all(t[k, :10] < 1.8e19) and t[k + 1, 1] < 1.8e19]
    if not ks:
        print("timeline: no complete iterations")
        return
    ph, lead = np.zeros(5), np.zeros(5)
    for k in ks:
        w = [t[k, 2 * i + 1] for i in range(5)] + [t[k + 1, 1]]
        for i in range(5):
            ph[i] += w[i + 1] - w[i]
            lead[i] += t[k, 2 * i + 1] - t[k, 2 * i]
    first = [k for k in range(0, min(iters, 256) - 1) if np.all(t[k, :10] < 1.8e19) and t[k + 1, 1] < 1.8e19][:12]
    print("proj phase of the first iterations (us):",
          " ".join(f"{(t[k, 3] - t[k, 1]) / 1e3:.0f}" for k in first))
    ph /= len(ks)
    lead /= len(ks)
    sub = {}
    for name, a, b in [("adj_finish tail start", 9, 10), ("adj_finish tail tree", 10, 15),
                       ("adj_finish tail scalar", 15, 11), ("adj_finish tail", 10, 11),
                       ("adj_tail -> next proj", 11, 17), ("fwd_finish tail start", 5, 12),
                       ("fwd_finish tail", 12, 13), ("fwd_tail -> adj", 13, 7),
                       ("proj body", 1, 14), ("proj end -> fwd_sparse", 14, 3)]:
        vals = []
        for k in ks:
            ta = t[k, a] if a < 16 else t[k + 1, a - 16]
            tb = t[k, b] if b < 16 else t[k + 1, b - 16]
            if ta < 1.8e19 and tb < 1.8e19 and tb > 0 and ta > 0:
                vals.append(tb - ta)
        if vals:
            sub[name] = np.median(vals) / 1e3
            if name == "adj_tail -> next proj":
                print("adj_tail -> next proj per iteration (us):",
                      " ".join(f"{v/1e3:.1f}" for v in vals[:24]))
    print("timeline details (median us): " + "  ".join(f"{k} {v:.2f}" for k, v in sub.items()))
    print(f"timeline over {len(ks)} iterations (us): " + "  ".join(
        f"{n} {p/1e3:.2f} (entered {l/1e3:.2f} early)" for n, p, l in zip(names, ph, lead)) +
        f"  | iteration {ph.sum()/1e3:.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--solves", type=int, default=1)
    ap.add_argument("--profile", action="store_true", help="print projection phase profile")
    ap.add_argument("--timing", action="store_true", help="per-kernel CUDA-event timing")
    ap.add_argument("--trace", action="store_true", help="print per-iteration support sizes")
    ap.add_argument("--clock-ghz", type=float, default=1.965)
    ap.add_argument("--timeline", action="store_true",
                    help="in-graph kernel start times per iteration (libl1g_tl.so)")
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
        if a.timeline:
            lib.l1g_debug_timeline_gemv(None, 1)
            lib.l1g_debug_timeline_proj(None, 1)
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
    if a.timeline:
        timeline(lib, res.iterations)
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
        out = (C.c_double * 32)()
        lib.l1g_solver_proj_profile(h, out)
        print("proj profile:", [round(v, 3) for v in out])
        calls = max(out[8], 1.0)
        names = {0: "steplength", 1: "v + |v|_1", 2: "michelot", 14: "count", 21: "hist atomics",
                 22: "hist gather", 15: "bins/bases", 16: "scatter", 17: "rank sort",
                 3: "gather", 5: "exact prefix", 6: "feasibility", 30: "h + stage",
                 31: "x,g loads, d, bitmap", 4: "g'd tree + block", 7: "exchange"}
        ghz = a.clock_ghz
        print("proj phases (us per call, CTA 0 clock at %.3f GHz): " % ghz + "  ".join(
            f"{nm} {out[i] / calls / ghz / 1e3:.2f}" for i, nm in names.items()) +
            f"  | total {sum(out[i] for i in names) / calls / ghz / 1e3:.2f}; michelot rounds "
            f"{out[10] / calls:.2f}, candidates {out[11] / calls:.0f}, bumps {out[12] / calls:.2f},"
            f" retries {out[13] / calls:.2f}, prefix epochs {out[20] / calls:.2f}")
        pn = {24: "head", 25: "pass1", 26: "tie segs", 27: "exchanges 1", 28: "pass2+events",
              29: "exchanges 2"}
        if any(out[i] for i in pn):
            print("cluster prefix (us per call): " + "  ".join(
                f"{nm} {out[i] / calls / ghz / 1e3:.2f}" for i, nm in pn.items()))
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
