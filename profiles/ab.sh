#!/bin/bash
# A/B of two builds of the product library on one GPU box: alternates the
# plain bench between paper_2012_14792_b200/libslicecraft_b200.so (B, current)
# and $1 (A, e.g. an older build copied in-tree), printing ms/step and phases.
A=${1:-paper_2012_14792_b200/libslicecraft_b200_prev.so}
ARGS=${2:-"--steps 10 --warmup 3 --no-cpu-baseline --no-extra"}
for i in 1 2 3; do
  for lib in "$A" paper_2012_14792_b200/libslicecraft_b200.so; do
    SLICECRAFT_B200_LIB=$PWD/$lib python bench.py $ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib'.split('/')[-1], round(d['ms_per_step'],4), d['phase_us'])"
  done
done
