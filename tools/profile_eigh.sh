#!/usr/bin/env bash
# Eigensolver evidence: per-phase sytrd cycle split and the launch list of
# three eigh(2048) calls (realistic FD-reduce size at C2).
set -u
OUT=${OUT:-gpurun_out}
AERO_SYTRD_PROF=1 timeout 300 python tools/time_eigh.py 2048 1024 512 256 > $OUT/eigh_prof.log 2>&1
echo "eigh prof rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/eigh_launches.csv python tools/time_eigh.py 2048 > $OUT/eigh_ncu.log 2>&1
echo "eigh launches rc=$?"
