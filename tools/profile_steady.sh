#!/usr/bin/env bash
# Steady-state C2 evidence: launch list over a window of the timed region and a
# --set full capture of three large k_product launches (rows > 24k).
set -u
OUT=${OUT:-gpurun_out}
CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 $CMD > $OUT/steady_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-40000} -c ${COUNT:-6000} --csv \
    --log-file $OUT/steady_launches.csv $CMD > $OUT/steady_ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_iterate} \
    -s ${KSKIP:-300} -c ${KCOUNT:-3} -o $OUT/steady_prof $CMD > $OUT/steady_ncu_full.log 2>&1
echo "full rc=$?"
