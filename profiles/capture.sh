#!/bin/bash
# GPU-box profiling recipe (run under gpurun from the repo root):
#   1. the plain bench (must exit 0 first), 2. the ncu launch list of the same
#   command, 3. one `ncu --set full` capture of the steady-state search walks
#   (step 1 + step 2 of one call) and of the texture kernel.
# Outputs go to gpurun_out/; profiles/summarize.py and profiles/launches.py
# turn them into the committed summaries.
set -e
TAG=${1:-prof}
CMD="python bench.py --steps 1 --warmup 3 --no-extra --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_search -s 4 -c 2 \
    -o gpurun_out/${TAG}_search $CMD > gpurun_out/${TAG}_search.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_texture -s 2 -c 1 \
    -o gpurun_out/${TAG}_texture $CMD > gpurun_out/${TAG}_texture.log 2>&1
echo captured
