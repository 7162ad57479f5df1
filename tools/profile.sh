#!/bin/bash
# Profiling recipe (run under gpurun, 1 GPU).  Writes into gpurun_out/.
#   1. plain run (must exit 0 before ncu touches the same command)
#   2. launch list with per-kernel device time (cold-cache, serialised)
#   3. one --set full capture of the sweep kernel
set -e
TAG=${1:-r01}
N=${N:-8192}
PREC=${PREC:-f64}
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --n $N --precision $PREC"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep -s 3 -c 1 \
    -o gpurun_out/${TAG}_sweep $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo profile done
