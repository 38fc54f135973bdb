"""Per-config divergence floor between equally legal reduction orders (VERDICT r1 "Next" #1).

The reference sums with Eigen's (unspecified, third-party) order; this repo fixes the
canonical pairwise order on both the GPU and the oracle.  How far can
two legal orders drift apart on each BASELINE problem?  For every config this tool runs the
same GPSS trajectory (gpss.cpp:221-292, x0 = 0, stationarity_tol = 0) three ways on the CPU:

  canonical  oracle/l1oracle.c, pairwise sums (== the GPU, bit for bit: tests/test_gpu_*parity)
  literal    the same oracle with plain sequential sums (O.LITERAL)
  fast       the reference's own sources (oracle/_ref/libref_fast.so: sequential sums)

and reports, canonical vs literal: relative ||dx|| and |df| at checkpoints, the first
iteration whose accepted steplength rule (bb_active) or backtracking halvings differ, the
first iteration whose support differs outside the 1e-12 band (coordinates where both
iterates are within 1e-12 of zero are not compared), and the comparison WINDOW: the last
iteration up to which every iterate and objective agree within 1e-9 (relative), the rule
and halvings agree and the supports agree.  `fast` is compared with `literal` record by
record (it should be the same arithmetic).

  python tools/divergence.py C1 C2mini C3mini C4mini C2 C3_300 C3 C5_0   -> profiles/r02_divergence.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402
from tests import problems as PB  # noqa: E402

SIGMA = json.load(open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")))
TOL = 1e-9
BAND = 1e-12


def c5_problem(j):
    """Problem j of C5 (BASELINE configs[4]) alone, built as harness.build_batch_problem does."""
    c = PB.C5_K
    n, p, seed, B = c["n"], c["p"], c["seed"], c["batch"]
    K = O.gaussian_matrix(seed, n, p)
    O.lib().orc_scale(K, K.size, 0.9 / SIGMA["C5"])
    sj = 1000 * seed + j
    spec = O.ProblemSpec("gaussian", n, p, c["nnz"], sj, "normal", c["noise"], "abs")
    x = np.zeros(p)
    x[O.sample_support(sj, 1, p, c["nnz"])] = O.x_true_values(spec, c["nnz"])
    with O.mode(O.CANONICAL):
        y = O.apply(K, x) + c["noise"] * O.fill_normal(sj, 2, 0, n)
        rho = (0.2 + 0.8 * j / (B - 1)) * O.l1norm(x)
    return K, y, rho


def problem(name):
    if name.startswith("C5_"):
        K, y, rho = c5_problem(int(name[3:]))
        return K, y, rho, 300
    base = name.split("_")[0]
    spec = {"C1": PB.C1, "C2": PB.C2, "C3": PB.C3, "C4": PB.C4, "C2mini": PB.C2_MINI,
            "C3mini": PB.C3_MINI, "C4mini": PB.C4_MINI}[base]
    iters = int(name.split("_")[1]) if "_" in name else PB.ITERS.get(base, {
        "C2mini": 300, "C3mini": 400, "C4mini": 200}.get(base, 300))
    if spec.kind == "gaussian" and base in SIGMA:
        import copy
        spec = copy.copy(spec)
        spec.sigma_hat = SIGMA[base]
    P = O.build_problem(spec)
    return P["K"], P["y"], P["rho"], iters


def support_differs(a, b):
    na, nb = a != 0.0, b != 0.0
    big = (np.abs(a) > BAND) | (np.abs(b) > BAND)
    return bool(np.any((na != nb) & big))


def run(name):
    t0 = time.time()
    K, y, rho, iters = problem(name)
    stop = O.StopRule(iters, 0, 0, 0.0)
    with O.mode(O.CANONICAL):
        xc, rc, recc, xhc = O.gpss_solve(K, y, rho, O.GpConfig(), stop, x_trace=True)
    with O.mode(O.LITERAL):
        xl, rl, recl, xhl = O.gpss_solve(K, y, rho, O.GpConfig(), stop, x_trace=True)
    out = {"n": int(K.shape[0]), "p": int(K.shape[1]), "iterations_cap": iters,
           "canonical": {"iterations": rc["iterations"], "reason": rc["reason_name"],
                         "objective": rc["objective"]},
           "literal": {"iterations": rl["iterations"], "reason": rl["reason_name"],
                       "objective": rl["objective"]}}
    kc = min(len(recc), len(recl))
    rel_dx, rel_df = [], []
    first_rule = first_halv = first_sup = None
    window = 0
    for i in range(kc):
        a, b = xhc[i], xhl[i]
        dx = float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-300))
        df = abs(recc[i]["f"] - recl[i]["f"]) / max(abs(recc[i]["f"]), 1e-300)
        rel_dx.append(dx)
        rel_df.append(df)
        if first_rule is None and recc[i]["bb_active"] != recl[i]["bb_active"]:
            first_rule = i + 1
        if first_halv is None and recc[i]["halvings"] != recl[i]["halvings"]:
            first_halv = i + 1
        if first_sup is None and support_differs(a, b):
            first_sup = i + 1
        if (window == i and dx <= TOL and df <= TOL and first_rule is None and
                first_halv is None and first_sup is None):
            window = i + 1
    cps = sorted(set([k for k in (10, 50, 100, 150, 200, 231, 250, 300, 400, 500, 1000, 1500,
                                  2000) if k <= kc] + ([kc] if kc else [])))
    out["checkpoints"] = {str(k): {"rel_dx": rel_dx[k - 1], "rel_df": rel_df[k - 1]}
                          for k in cps}
    out["max_rel_dx_common"] = max(rel_dx) if rel_dx else 0.0
    out["first_rule_mismatch"] = first_rule
    out["first_halvings_mismatch"] = first_halv
    out["first_support_mismatch"] = first_sup
    out["window"] = window
    out["final_rel_dx"] = float(np.linalg.norm(xc - xl) / max(np.linalg.norm(xc), 1e-300))
    out["final_abs_df"] = abs(rc["objective"] - rl["objective"])
    if R.available("fast") and K.nbytes <= 32 << 30:  # C4: no room for the column-major copy
        xf, rf, recf = R.RefOperator(K, "fast").gpss_solve(y, rho, O.GpConfig(), stop)
        same_recs = len(recf) == len(recl) and all(
            all((a[f] == b[f]) or (np.isnan(a[f]) and np.isnan(b[f]))
                for f in ("f", "alpha", "step", "bb_active", "bb1_raw", "bb2_raw", "f_max"))
            for a, b in zip(recf, recl))
        out["fast_vs_literal"] = {"iterations": rf["iterations"],
                                  "records_bit_identical": bool(same_recs),
                                  "x_bit_identical": bool(np.array_equal(xf, xl)),
                                  "rel_dx_vs_canonical": float(np.linalg.norm(xf - xc) /
                                                               max(np.linalg.norm(xc), 1e-300))}
    out["seconds"] = round(time.time() - t0, 1)
    return out


def main(names):
    path = os.path.join(ROOT, "profiles", "r02_divergence.json")
    allres = json.load(open(path)) if os.path.exists(path) else {}
    for nm in names:
        allres[nm] = run(nm)
        print(nm, json.dumps(allres[nm]), flush=True)
        with open(path, "w") as f:
            json.dump(allres, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2mini", "C3mini", "C4mini"])
