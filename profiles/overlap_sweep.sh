#!/bin/bash
# Sweep of the texture-pass overlap knobs on the headline bench: trace-walk
# blocks per SM (room for K1 blocks beside step 1) x K1 enqueued before or
# after the time tables.
for cfg in "" "SLICECRAFT_B200_TRACE_BPS=7" "SLICECRAFT_B200_TRACE_BPS=7 SLICECRAFT_B200_K1_LATE=1" \
           "SLICECRAFT_B200_TRACE_BPS=6 SLICECRAFT_B200_K1_LATE=1" "SLICECRAFT_B200_K1_LATE=1"; do
  env $cfg python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('[$cfg]', round(d['ms_per_step'],4), d['phase_us'])"
done
