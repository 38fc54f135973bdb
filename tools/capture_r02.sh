#!/bin/bash
# ncu evidence for profiles/ (round 2).  Every ncu command runs after the same command line
# exited 0 without ncu (the recipe in B200_PROFILING.md).  Then, here:
#   python tools/write_profiles_r02.py
# Usage on the GPU box: bash tools/capture_r02.sh [what...]   (default: all)
set -x
mkdir -p gpurun_out
O=gpurun_out
what="${*:-c4launch c4full c2full c2launch c5full c5launch}"
for w in $what; do
case $w in
c4launch)  # the bench default (C4): every launch of one timed solve, cold-cache, serialised
  python tools/prof_solve.py --config C4 --iters 12 > $O/plain_c4.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_c4.csv \
      python tools/prof_solve.py --config C4 --iters 12 > $O/ncu_launch_c4.log 2>&1
  ;;
c4full)  # one launch of each iteration kernel at C4 (iteration 8 of 10)
  python tools/prof_solve.py --config C4 --iters 10 > $O/plain_c4f.log 2>&1 &&
  ncu --set full --import-source on --clock-control none \
      -k regex:"adj_kernel|fwd_sparse|proj_kernel|fwd_finish|adj_finish" -s 40 -c 5 \
      -o $O/full_c4 -f python tools/prof_solve.py --config C4 --iters 10 > $O/ncu_full_c4.log 2>&1
  ;;
c2full)
  python tools/prof_solve.py --config C2 --iters 60 > $O/plain_c2f.log 2>&1 &&
  ncu --set full --import-source on --clock-control none \
      -k regex:"adj_kernel|fwd_sparse|proj_kernel|fwd_finish|adj_finish" -s 200 -c 5 \
      -o $O/full_c2 -f python tools/prof_solve.py --config C2 --iters 60 > $O/ncu_full_c2.log 2>&1
  ;;
c2launch)
  python tools/prof_solve.py --config C2 --iters 80 > $O/plain_c2l.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_c2.csv \
      python tools/prof_solve.py --config C2 --iters 80 > $O/ncu_launch_c2.log 2>&1
  ;;
c5full)
  python tools/prof_batch.py --iters 5 --solves 1 > $O/plain_c5f.log 2>&1 &&
  ncu --set full --import-source on --clock-control none -k regex:"bfwd|badj|proj_kernel|bfin" \
      -s 12 -c 6 -o $O/full_c5 -f python tools/prof_batch.py --iters 5 --solves 1 > $O/ncu_full_c5.log 2>&1
  ;;
c5launch)
  python tools/prof_batch.py --iters 20 --solves 1 > $O/plain_c5l.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launch_c5.csv \
      python tools/prof_batch.py --iters 20 --solves 1 > $O/ncu_launch_c5.log 2>&1
  ;;
esac
done
ls -la $O
