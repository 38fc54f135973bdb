import sys, ctypes as C, numpy as np
sys.path.insert(0, "/root/repo")
import paper_0902_4424_b200 as l1
from paper_0902_4424_b200 import _lib as L
from tests.test_gpu_batch import batch_problems
for (n, p, B) in [(200, 2048, 16), (1024, 4096, 16), (512, 2048, 16)]:
    K, Y, rho = batch_problems(n, p, B, 31 + B)
    op = l1.DenseOperator(K)
    lib = L.load()
    for iters in (10, 20, 40, 80, 160):
        cfg = l1.GpConfig()._c(); stop = l1.StopRule(max_iterations=iters, stationarity_tol=0.0)._c()
        X = np.empty((B, p)); res = (L.ResultC * B)()
        L.check(lib.l1g_gpss_solve_batched(op.h, B, L.ptr(np.ascontiguousarray(Y)), L.ptr(rho), C.byref(cfg), C.byref(stop), L.ptr(X), res))
        devs = []
        for b in range(B):
            sol = l1.gpss_solve(l1.Objective(op, Y[b]), l1.L1Ball(rho[b]), l1.GpConfig(), l1.StopRule(max_iterations=iters, stationarity_tol=0.0))
            devs.append((np.abs(X[b]-sol.x).max()/max(1,np.abs(sol.x).max()), res[b].iterations, sol.iterations, int(sol.reason)))
        worst = max(devs)
        print(n, p, B, iters, "worst rel dev %.2e" % worst[0], "iters", worst[1:], "n>1e-9:", sum(d[0] > 1e-9 for d in devs), flush=True)
