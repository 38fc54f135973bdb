"""Batched solves with the products on the compacted live problems against the in-place full-width
products, bit for bit, over several (n, p, B) incl. B = 1, partial and multiple problem blocks
(each variant in its own process: the switch is read once).  python tools/batch_compaction_check.py"""
import os, subprocess, sys, numpy as np
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SN = r"""
import ctypes as C, sys, numpy as np
sys.path.insert(0, {root!r})
import paper_0902_4424_b200 as l1
from paper_0902_4424_b200 import _lib as L
from tests.test_gpu_batch import batch_problems
n, p, B, seed, iters = {n}, {p}, {B}, {seed}, {iters}
K, Y, rho = batch_problems(n, p, B, seed)
op = l1.DenseOperator(K)
lib = L.load()
cfg = l1.GpConfig(memory={mem})._c()
stop = l1.StopRule(max_iterations=iters, stationarity_tol=0.0)._c()
X = np.empty((B, p))
res = (L.ResultC * B)()
L.check(lib.l1g_gpss_solve_batched(op.h, B, L.ptr(np.ascontiguousarray(Y)), L.ptr(rho),
                                   C.byref(cfg), C.byref(stop), L.ptr(X), res), "batched")
np.savez({out!r}, X=X, its=np.array([res[b].iterations for b in range(B)]),
         f=np.array([res[b].objective for b in range(B)]))
"""
bad = 0
for (n, p, B, iters, mem) in [(100, 500, 129, 300, 1), (300, 1000, 300, 300, 1), (64, 4096, 257, 120, 3),
                              (512, 512, 33, 300, 1), (1024, 2048, 8, 300, 1), (96, 300, 1, 200, 1),
                              (200, 2048, 385, 200, 5)]:
    outs = []
    for name, env in [("plain", {"L1G_BATCH_COMPACT": "0"}), ("compact", {"L1G_BATCH_COMPACT": "1"})]:
        out = f"/tmp/bf_{name}.npz"
        r = subprocess.run([sys.executable, "-c", SN.format(root=root, out=out, n=n, p=p, B=B, seed=n + B, iters=iters, mem=mem)],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-1500:]
        outs.append(np.load(out))
    a, b = outs
    same = np.array_equal(a["its"], b["its"]) and np.array_equal(a["f"], b["f"]) and np.array_equal(a["X"], b["X"])
    print((n, p, B), "iterations", int(a["its"].min()), int(a["its"].max()), "identical" if same else "MISMATCH", flush=True)
    bad += not same
sys.exit(bad)
