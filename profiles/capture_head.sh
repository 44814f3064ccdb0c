#!/bin/bash
# GPU-box recipe: the plain bench (must exit 0 first), then one `ncu --set
# full` capture (with source) of one steady-state kernel (default the
# exhaustive step-1 walk; arg 2 = kernel regex) and the launch list of the
# same command.  Outputs under
# gpurun_out/<TAG>_*; read here with ncu -i ... --page source --csv.
set -e
TAG=${1:-head}
KERNEL=${2:-k_search_head}
CMD="python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
ncu --set full --clock-control none --import-source on -k regex:$KERNEL -s 2 -c 1 \
    -o gpurun_out/${TAG}_head $CMD > gpurun_out/${TAG}_head.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
echo captured
