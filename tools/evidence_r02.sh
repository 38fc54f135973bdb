#!/bin/bash
# Round-2 evidence on one B200: benches of every config, projection phases, in-graph timeline,
# forward crossover, then the ncu captures (tools/capture_r02.sh).  Afterwards, here:
#   python tools/write_profiles_r02.py
set -x
O=gpurun_out
if [ -n "$ONLY_FULL" ]; then bash tools/capture_r02.sh c4full c2full c5full; exit; fi
mkdir -p $O
timeout 900 python bench.py > $O/ev_bench_C4.json 2> $O/ev_bench_C4.err
for c in C2 C5 C1; do timeout 600 python bench.py --config $c --steps 10 > $O/ev_bench_$c.json 2> $O/ev_bench_$c.err; done
timeout 900 python bench.py --config C3 --steps 3 > $O/ev_bench_C3.json 2> $O/ev_bench_C3.err
for c in C2 C4; do python tools/prof_solve.py --config $c --iters 80 --solves 2 --profile > $O/ev_phases_$c.txt 2>&1; done
python tools/prof_solve.py --config C2 --iters 80 --solves 2 --timeline > $O/ev_timeline_C2.txt 2>&1
python tools/prof_solve.py --config C4 --iters 30 --solves 2 --timeline > $O/ev_timeline_C4.txt 2>&1
python tools/fwd_crossover.py > $O/ev_crossover_C2.txt 2>&1
bash tools/capture_r02.sh ${CAPTURE:-c4launch c2launch c5launch}
