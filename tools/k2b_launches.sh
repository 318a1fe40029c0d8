#!/usr/bin/env bash
# Kernel launch list of one config-5 window factorization (K2b), for the time split.
set -o pipefail
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/k2b_launches.csv python tools/cfg5_full.py factor_rate --batch 1 \
    --out gpurun_out/k2b_ncu.jsonl > gpurun_out/k2b_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/k2b_launches.csv | head -30
