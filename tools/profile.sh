#!/bin/bash
# GPU-box profiling recipe (run under gpurun from the repo root):
#   tools/profile.sh <tag> [bench args...]
# 1. launch list of one bench run (cold, serialised per-kernel device times)
# 2. ncu --set full of every kernel of the 3rd warm-up search (skip the first
#    two searches, capture the next 40 launches)
# Outputs land in gpurun_out/<tag>_*.
set -u
tag=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu "$@" \
    > gpurun_out/${tag}_launches.log 2>&1
# 1b. the same with caches left warm (L2 state as the previous kernel left it)
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_launches_warm.csv python bench.py --steps 2 --warmup 3 --no-cpu "$@" \
    > gpurun_out/${tag}_launches_warm.log 2>&1
ncu --set full --clock-control none --import-source on -s 38 -c 40 \
    -o gpurun_out/${tag}_full -f python bench.py --steps 1 --warmup 3 --no-cpu "$@" \
    > gpurun_out/${tag}_full.log 2>&1
tail -2 gpurun_out/${tag}_full.log
