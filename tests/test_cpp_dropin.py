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
