#!/usr/bin/env bash
# Config-size covariance-error runs (tools/full_run.py) for the given configs.
set -u
mkdir -p gpurun_out
for c in "$@"; do
  timeout 1500 python tools/full_run.py --config $c --out gpurun_out/full_$c.json > gpurun_out/full_$c.log 2>&1
  echo "$c rc=$?" >> gpurun_out/full_runs.rc
done
