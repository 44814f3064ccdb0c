#!/bin/bash
# Round-2 captures (run under gpurun from the repo root): the plain bench
# first, then the ncu launch list of the same command, one `ncu --set full`
# capture of the step-1 trace walk, of K1, and of the step-2 trace walk on
# the covering family at lambda 0.3 (where it is the chosen step-2 walk).
set -e
TAG=${1:-r02}
CMD="python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trace_walk -s 2 -c 1 \
    -o gpurun_out/${TAG}_search $CMD > gpurun_out/${TAG}_search.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_texture -s 2 -c 1 \
    -o gpurun_out/${TAG}_texture $CMD > gpurun_out/${TAG}_texture.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_trace_walk2 -s 3 -c 1 \
    -o gpurun_out/${TAG}_step2cov python bench.py --steps 1 --warmup 4 --no-extra \
    --no-cpu-baseline --lambda 0.3 --coverage 1 > gpurun_out/${TAG}_step2cov.log 2>&1
echo captured
