#!/bin/bash
# usage: tools/launches.sh <config> <tag>  — ncu launch list (gpu__time_duration) of one pipeline pass
cfg=${1:-c2}; tag=${2:-x}
python tools/ncu_target.py $cfg > gpurun_out/p_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python tools/ncu_target.py $cfg > gpurun_out/n_$tag.log 2>&1
