#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box after the same commands exited 0 without ncu).
#   cold launch lists (recipe: gpu__time_duration.sum, --clock-control none, caches flushed),
#   warm launch lists (--cache-control none: closer to the in-graph durations), and one
#   --set full capture per hot kernel.  Then, here: python tools/write_profiles.py
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launch_c2_warm.csv \
    python tools/prof_solve.py --config C2 --iters 80 > gpurun_out/ncu_launch_c2_warm.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"adj_kernel|fwd_sparse|proj_kernel|fwd_finish|adj_finish" \
    -s 200 -c 5 -o gpurun_out/full_c2 -f python tools/prof_solve.py --config C2 --iters 60 > gpurun_out/ncu_full_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"bfwd|badj|proj_kernel|bfin" -s 12 -c 6 \
    -o gpurun_out/full_c5 -f python tools/prof_batch.py --iters 5 --solves 1 > gpurun_out/ncu_full_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5.csv \
    python tools/prof_batch.py --iters 20 --solves 1 > gpurun_out/ncu_launch_c5.log 2>&1
# in-graph kernel timeline (debug build with %globaltimer stamps, not a profiler)
python tools/prof_solve.py --config C2 --iters 80 --solves 2 --timeline > gpurun_out/timeline_c2.txt 2>&1
python tools/prof_solve.py --config C2 --iters 80 --solves 2 --profile > gpurun_out/proj_phases_c2.txt 2>&1
ls -la gpurun_out
