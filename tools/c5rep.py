import ctypes as C, json, os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_0902_4424_b200 as l1
from paper_0902_4424_b200 import _lib as L, harness as H
SIG = json.load(open("tests/golden/sigma_hat.json"))
c = dict(H.C5)
P = H.build_batch_problem(**c, sigma_hat=SIG["C5"])
B, p = c["batch"], c["p"]
for rep in range(int(sys.argv[1])):
    X = np.empty((B, p)); res = (L.ResultC * B)()
    try:
        L.check(L.load().l1g_gpss_solve_batched(P["op"].h, B, L.ptr(np.ascontiguousarray(P["Y"])), L.ptr(P["rho"]),
            C.byref(l1.GpConfig()._c()), C.byref(l1.StopRule(max_iterations=int(sys.argv[2]), stationarity_tol=0.0)._c()), L.ptr(X), res))
        print(rep, "ok", res[0].iterations, flush=True)
    except Exception as e:
        print(rep, "FAIL", e, flush=True); break
