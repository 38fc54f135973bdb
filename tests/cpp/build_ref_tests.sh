#!/usr/bin/env bash
# Compiles the reference's own unit tests -- /root/reference/proj/tests/test_{gpss,prox,
# solvers}.cpp and test_main.cpp, read in place and unchanged -- against this repo's drop-in
# headers (include/l1solve) and libraries (libl1solve_b200.so -> libl1g.so), with a doctest
# stand-in (tests/cpp/doctest_shim).  The binary goes to tests/cpp/_ref/ (git-ignored; it
# travels to the GPU box, which has no /root/reference) and is run by
# tests/test_cpp_dropin.py::test_reference_unit_tests_pass.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${L1_REFERENCE:-/root/reference}/proj/tests"
OUT="$HERE/_ref"
if [ ! -f "$REF/test_gpss.cpp" ]; then
  echo "reference tests not found at $REF; skipping" >&2
  exit 0
fi
mkdir -p "$OUT"
PKG="$ROOT/paper_0902_4424_b200"
CXX="${L1_REF_CXX:-/usr/bin/g++}"
$CXX -std=c++17 -O1 -ffp-contract=off -I"$ROOT/include" -I"$HERE/doctest_shim" -I"$REF" \
  "$REF/test_main.cpp" "$REF/test_gpss.cpp" "$REF/test_prox.cpp" "$REF/test_solvers.cpp" \
  -o "$OUT/ref_unit_tests" -L"$PKG" -l:libl1solve_b200.so -l:libl1g.so -Wl,-rpath,"$PKG"
echo "built $OUT/ref_unit_tests"
