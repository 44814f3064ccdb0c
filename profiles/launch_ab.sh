#!/bin/bash
# Launch lists (ncu gpu__time_duration, cold + serialised) of the plain bench
# under two builds of the product library: A = $1, B = the current build.
A=${1:-paper_2012_14792_b200/libslicecraft_b200_prev.so}
TAG=${2:-ab}
CMD="python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-extra"
for which in A B; do
  lib=$PWD/paper_2012_14792_b200/libslicecraft_b200.so
  [ $which = A ] && lib=$PWD/$A
  SLICECRAFT_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_${which}.csv $CMD > /dev/null 2>&1
done
echo done
