"""cond(K) of the C3 blur operator (BASELINE.json configs[2]): K is the
symmetric banded Toeplitz matrix of unit-sum Gaussian taps (sigma = 4 samples, radius 12 =
3 sigma, zero boundary), so all eigenvalues come from LAPACK's banded symmetric solver and
cond_2(K) = max|lambda| / min|lambda|.  Writes profiles/c3_condition.json."""
import json
import os
import sys

import numpy as np
from scipy.linalg import eigvals_banded

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

out = {}
taps = O.blur_taps()
R = O.BLUR_RADIUS
for n in (1024, 2048, 16384):
    band = np.zeros((R + 1, n))  # upper form: band[R - k, j] = K[j - k, j]
    for k in range(R + 1):
        band[R - k, k:] = taps[R + k]
    ev = eigvals_banded(band, lower=False)
    a = np.abs(ev)
    out[str(n)] = {"sigma_max": float(a.max()), "sigma_min": float(a.min()),
                   "cond": float(a.max() / a.min())}
    print(n, out[str(n)])
json.dump(out, open(os.path.join(ROOT, "profiles", "c3_condition.json"), "w"), indent=1)
