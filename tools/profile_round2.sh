#!/usr/bin/env bash
# Round-2 evidence for profiles/ (one GPU, after the same command exited 0
# without ncu): (a) launch list of the default C2 bench command, (b) one
# --set full capture of the dominant kernel k_iterate_i8 in steady state,
# (c) duration + DRAM bytes of every GEMM / ingest / copy launch (HBM GB/s of
# the append Gram block and the reduce rotation).
set -u
OUT=${OUT:-gpurun_out}
CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu"
timeout 900 $CMD > $OUT/r2_plain.json 2> $OUT/r2_plain.err || { echo "plain run failed"; exit 1; }
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 400000 --csv \
    --log-file $OUT/r2_launches.csv $CMD > $OUT/r2_ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_iterate_i8 \
    -s ${KSKIP:-400} -c 2 -o $OUT/r2_k_iterate_i8 $CMD > $OUT/r2_ncu_full.log 2>&1
echo "full rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'k_product_mma|k_ingest|k_copy_matrix|k_sytrd_rows' -c 400000 --csv \
    --log-file $OUT/r2_hbm.csv $CMD > $OUT/r2_ncu_hbm.log 2>&1
echo "hbm rc=$?"
