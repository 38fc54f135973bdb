"""Build recipe for libl1g.so (sm_100a only)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["gemv.cu", "dmma.cu", "project.cu", "small.cu", "vec.cu", "comm.cu", "abi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-fmad=false", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-ldl"]


def lib_path():
    return os.path.join(HERE, "libl1g.so")


def dropin_path():
    return os.path.join(HERE, "libl1solve_b200.so")


INCLUDE = os.path.join(HERE, "..", "include")
CXX = os.environ.get("L1G_CXX", "/usr/bin/g++")


def build_dropin(verbose=False):
    """The reference's C++ API (include/l1solve/*.hpp) over the C-ABI."""
    cmd = [CXX, "-std=c++17", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
           f"-I{INCLUDE}", os.path.join(CSRC, "l1solve_dropin.cpp"), "-o", dropin_path(),
           f"-L{HERE}", "-l:libl1g.so", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return dropin_path()


def needs_build():
    out = lib_path()
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "l1g.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile_link(out: str, defines: list[str], verbose: bool):
    """One nvcc per source file, run side by side, then one link."""
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    cflags = [f for f in FLAGS if f not in ("-shared", "-cudart", "static", "-ldl")]
    with tempfile.TemporaryDirectory(prefix="l1g_build_") as tmp:
        objs = [os.path.join(tmp, s.replace(".cu", ".o")) for s in SOURCES]
        cmds = [[NVCC, *cflags, *defines, "-c", os.path.join(CSRC, s), "-o", o]
                for s, o in zip(SOURCES, objs)]
        if verbose:
            for c in cmds:
                print(" ".join(c))
        with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
            for r in ex.map(lambda c: subprocess.run(c), cmds):
                if r.returncode != 0:
                    raise subprocess.CalledProcessError(r.returncode, r.args)
        link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared",
                "-cudart", "static", "-ldl", "-o", out, *objs]
        if verbose:
            print(" ".join(link))
        subprocess.run(link, check=True)


def build(force: bool = False, verbose: bool = False):
    if not force and not needs_build():
        return lib_path()
    _compile_link(lib_path(), [], verbose)
    build_dropin(verbose)
    return lib_path()


def build_variant(name: str, defines: list[str], verbose: bool = False) -> str:
    """Debug variants (e.g. -DL1G_TIMELINE) as lib<name>.so next to libl1g.so; loaded through
    L1G_LIB_PATH by the profiling tools only."""
    out = os.path.join(HERE, f"lib{name}.so")
    _compile_link(out, defines, verbose)
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
