#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box after the same commands exited 0 without ncu).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1
ncu --set full --import-source on -k regex:"adj_kernel|fwd_sparse|proj_kernel|fwd_finish|adj_finish" \
    -s 40 -c 5 -o gpurun_out/full_c2 python tools/prof_solve.py --config C2 --iters 30 > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --import-source on -k regex:"bfwd|badj" -c 2 -o gpurun_out/full_c5 \
    python tools/prof_batch.py --iters 3 --solves 1 > gpurun_out/ncu_full_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5.csv \
    python tools/prof_batch.py --iters 20 --solves 1 > gpurun_out/ncu_launch_c5.log 2>&1
