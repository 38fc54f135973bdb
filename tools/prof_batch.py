"""Time a batched (C5-shaped) solve: python tools/prof_batch.py [--iters 300] [--batch 128]"""
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

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=300)
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--solves", type=int, default=2)
a = ap.parse_args()
fx = json.load(open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")))
c = dict(H.C5)
c["batch"] = a.batch
P = H.build_batch_problem(**c, sigma_hat=fx.get("C5"))
lib = L.load()
B, n, p = a.batch, c["n"], c["p"]
h = C.c_void_p()
cfg = l1.GpConfig()._c()
L.check(lib.l1g_batch_create(P["op"].h, B, L.ptr(np.ascontiguousarray(P["Y"])), L.ptr(P["rho"]),
                             C.byref(cfg), C.byref(h)))
stop = l1.StopRule(max_iterations=a.iters, stationarity_tol=0.0)._c()
res = (L.ResultC * B)()
for s in range(a.solves):
    t = time.perf_counter()
    L.check(lib.l1g_batch_init(h, None))
    L.check(lib.l1g_batch_run(h, C.byref(stop), res))
    dt = time.perf_counter() - t
    its = [res[i].iterations for i in range(B)]
    print(f"solve {s}: {dt*1e3:.1f} ms, max iterations {max(its)}, min {min(its)}, "
          f"{max(its)/dt:.1f} lockstep it/s, {sum(its)/dt:.0f} problem-it/s, "
          f"{4.0*n*p*B*max(its)/dt/1e12:.1f} TFLOP/s (4npB per lockstep iteration)", flush=True)
if os.environ.get("L1G_PRINT_LIVE"):
    live = [sum(1 for v in its if v > k) for k in range(max(its))]
    print("live problems per lockstep iteration:", live)
    print("live 32-groups after compaction:", [(v + 31) // 32 for v in live])
lib.l1g_batch_destroy(h)
