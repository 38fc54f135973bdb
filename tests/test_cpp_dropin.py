"""The C++ drop-in API (include/l1solve/*.hpp -> libl1solve_b200.so -> libl1g.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_0902_4424_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")


def compile_test(tmp_path):
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-ffp-contract=off",
                    f"-I{os.path.join(ROOT, 'include')}", SRC, "-o", exe, f"-L{PKG}",
                    "-l:libl1solve_b200.so", "-l:libl1g.so", f"-Wl,-rpath,{PKG}"], check=True)
    return exe


def test_dropin_compiles_and_links(tmp_path):
    """Headers compile and every symbol resolves against the built libraries (no GPU)."""
    assert os.path.exists(os.path.join(PKG, "libl1solve_b200.so"))
    compile_test(tmp_path)


@pytest.mark.gpu
def test_dropin_runs(tmp_path):
    exe = compile_test(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


REF_TESTS = os.path.join(ROOT, "tests", "cpp", "_ref", "ref_unit_tests")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/tests"),
                    reason="reference checkout absent (GPU box)")
def test_reference_unit_tests_compile_unchanged():
    """/root/reference/proj/tests/test_{gpss,prox,solvers}.cpp, unchanged, compile and link
    against include/l1solve + libl1solve_b200.so (tests/cpp/build_ref_tests.sh)."""
    subprocess.run([os.path.join(ROOT, "tests", "cpp", "build_ref_tests.sh")], check=True)
    assert os.path.exists(REF_TESTS)


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference unit tests not built")
def test_reference_unit_tests_pass():
    """The reference's own unit tests (53 test cases of test_gpss / test_prox / test_solvers)
    run on the GPU through the drop-in and pass."""
    r = subprocess.run([REF_TESTS], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
