"""Generates tests/golden/sigma_hat.json: the power-iteration estimate
spectral_norm_estimate(K_raw, 1000, 1e-8) (linear_operator.cpp:43-60) of the raw Gaussian
operators of the BASELINE configs, computed on the B200 with the canonical reductions.
tests/test_gpu_parity.py::test_spectral_norm_bit_identical pins the device power iteration
bit-for-bit to the CPU oracle at sizes the oracle can run; at full size the CPU would need
hours, so the reference arm and the sharded runs read this fixture.
Run on a GPU box:  python tests/golden/make_sigma.py C2 C4 C5
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_0902_4424_b200 as l1  # noqa: E402
from paper_0902_4424_b200 import harness as H  # noqa: E402

SHAPES = {k: (v.n, v.p, v.seed) for k, v in H.CONFIGS.items() if v.kind == "gaussian"}
SHAPES["C5"] = (4096, 16384, 5)


def main(names):
    path = os.path.join(ROOT, "tests", "golden", "sigma_hat.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for nm in names:
        n, p, seed = SHAPES[nm]
        t = time.time()
        op = l1.DenseOperator.generate_gaussian(n, p, seed)
        mv = l1.MatvecCounter()
        s = l1.spectral_norm_estimate(op, 1000, 1e-8, mv)
        out[nm] = s
        out[nm + "_matvecs"] = mv.count
        print(nm, repr(s), mv.count, f"{time.time() - t:.1f}s", flush=True)
        op.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "sigma_hat.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2", "C5", "C4"])
