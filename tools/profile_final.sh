#!/usr/bin/env bash
# Round-end evidence for profiles/: launch list (per-kernel device times) of
# the whole default C2 bench command at --steps 1 --warmup 3 (the summary
# keeps the last quarter = the timed step), after the same command exited 0
# without ncu.
set -u
OUT=${OUT:-gpurun_out}
CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 $CMD > $OUT/final_plain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 200000 --csv \
    --log-file $OUT/final_launches.csv $CMD > $OUT/final_ncu_launches.log 2>&1
echo "launch list rc=$?"
