"""L1PROBv1 problem files (problem_io.cpp) through the device path: byte-identical files,
the same FNV-1a hash as the oracle (pinned to the reference in tests/test_oracle_ref.py)."""
import numpy as np
import pytest

import paper_0902_4424_b200 as l1
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p", [(3, 4), (77, 301), (100, 262144)])
def test_load_save_hash(tmp_path, n, p):
    rng = np.random.default_rng(n + p)
    K = rng.normal(size=(n, p))
    y, x = rng.normal(size=n), rng.normal(size=p) * (rng.random(p) < 0.05)
    seed, noise = 123456789012345, 0.0125
    src = tmp_path / "src.l1prob"
    O.save_problem(src, K, y, x, seed, noise)
    prob = l1.load_problem(src)
    assert prob.seed == seed and prob.noise_level == noise
    assert np.array_equal(prob.y, y) and np.array_equal(prob.x_true, x)
    assert np.array_equal(prob.op.matrix(), K)
    assert l1.problem_hash(prob) == O.problem_hash(K, y, x, seed, noise)
    out = tmp_path / "out.l1prob"
    l1.save_problem(prob, out)
    assert out.read_bytes() == src.read_bytes()
    # the loaded operator computes like one built from K
    v = rng.normal(size=p)
    assert np.array_equal(prob.op.apply(v), O.apply(K, v))


def test_generated_operator_round_trip(tmp_path):
    op = l1.DenseOperator.generate_gaussian(64, 512, 7)
    y, x = np.arange(64.0), np.zeros(512)
    prob = l1.GeneratedProblem(op, y, x, 0.5, 7)
    path = tmp_path / "g.l1prob"
    l1.save_problem(prob, path)
    back = l1.load_problem(path)
    assert np.array_equal(back.op.matrix(), op.matrix())
    assert l1.problem_hash(back) == l1.problem_hash(prob)


def test_bad_files(tmp_path):
    bad = tmp_path / "bad.l1prob"
    bad.write_bytes(b"NOTAPROB" + bytes(64))
    with pytest.raises(RuntimeError):
        l1.load_problem(bad)
    O.save_problem(tmp_path / "t.l1prob", np.ones((4, 5)), np.ones(4), np.ones(5), 1, 0.0)
    raw = (tmp_path / "t.l1prob").read_bytes()
    (tmp_path / "short.l1prob").write_bytes(raw[:-8])
    with pytest.raises(RuntimeError):
        l1.load_problem(tmp_path / "short.l1prob")
    with pytest.raises(RuntimeError):
        l1.load_problem(tmp_path / "missing.l1prob")
