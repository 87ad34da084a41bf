#!/bin/bash
# ncu launch list of a short bench run (after a plain run of the same command): per-kernel summary
# usage (under gpurun): bash tools/launches.sh <tag> [bench args]
tag=$1; shift
python bench.py --profile --steps 3 --warmup 3 "$@" > gpurun_out/plain_$tag.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --profile --steps 3 --warmup 3 "$@" > gpurun_out/ncu_$tag.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$tag.csv | head -${LINES_SHOWN:-16}
