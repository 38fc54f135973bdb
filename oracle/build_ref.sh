#!/usr/bin/env bash
# Compiles the reference's own hot-path sources (read in place from /root/reference, never
# copied) against oracle/eigen_shim into oracle/_ref/.  Eigen itself is absent from the
# image, so the shim supplies the linear algebra; see oracle/eigen_shim/Eigen/Core.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${L1_REFERENCE:-/root/reference}/proj/core"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not found at $REF; skipping oracle/_ref" >&2
  exit 0
fi
mkdir -p "$OUT"
SRCS="$REF/src/gpss.cpp $REF/src/prox.cpp $REF/src/linear_operator.cpp $REF/src/objective.cpp $REF/src/psd.cpp $REF/src/shrinkage.cpp $REF/src/problem_io.cpp $REF/src/reference.cpp $HERE/ref_capi.cpp"
CXX="${L1_REF_CXX:-/usr/bin/g++}"
COMMON="-std=c++20 -fPIC -shared -ffp-contract=off -fno-fast-math -I$HERE/eigen_shim -I$REF/include"
# OpenMP splits GEMV outputs over threads only: the canonical values do not depend on it
$CXX -O2 -fopenmp $COMMON -o "$OUT/libref_canon.so" $SRCS
$CXX -O3 -fopenmp -DL1SHIM_FAST $COMMON -o "$OUT/libref_fast.so" $SRCS
echo "built $OUT/libref_canon.so $OUT/libref_fast.so"
