#!/usr/bin/env bash
# ncu evidence for profiles/: launch list (per-kernel device times) and one
# --set full capture of the dominant kernel. Run on the GPU box via gpurun.
set -u
OUT=${OUT:-gpurun_out}
CMD="python bench.py --config ${CFG:-c2} --steps 1 --warmup 1 --rows-per-step ${RPS:-2048} --no-e2e --no-cpu"
timeout 600 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-2000} -c ${COUNT:-4000} --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_product} -s ${KSKIP:-300} -c 3 \
    -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
