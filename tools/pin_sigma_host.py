"""Pins the committed sigma_hat fixture (tests/golden/sigma_hat.json, made on the B200) to the
CPU oracle at full size: spectral_norm_estimate(K_raw, 1000, 1e-8) (linear_operator.cpp:43-60)
recomputed on the host with the OpenMP oracle (order-preserving, canonical reductions).
Writes profiles/sigma_pin_host.json.  Usage: python tools/pin_sigma_host.py C2 C5 [C4]
(C4 needs ~70 GB of host RAM)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

SHAPES = {"C2": (8192, 32768, 2), "C4": (32768, 262144, 4), "C5": (4096, 16384, 5)}


def main(names):
    fix = json.load(open(os.path.join(ROOT, "tests", "golden", "sigma_hat.json")))
    path = os.path.join(ROOT, "profiles", "sigma_pin_host.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for nm in names:
        n, p, seed = SHAPES[nm]
        t = time.time()
        K = O.gaussian_matrix(seed, n, p)
        with O.mode(O.CANONICAL):
            s, mv = O.spectral_norm(K, 1000, 1e-8)
        out[nm] = {"host_sigma_hat": s, "host_matvecs": mv, "fixture": fix.get(nm),
                   "fixture_matvecs": fix.get(nm + "_matvecs"),
                   "bit_identical": s == fix.get(nm) and mv == fix.get(nm + "_matvecs"),
                   "seconds": round(time.time() - t, 1), "threads": os.cpu_count()}
        print(nm, out[nm], flush=True)
        del K
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C5", "C2"])
