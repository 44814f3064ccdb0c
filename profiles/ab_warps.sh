# A/B of the step-1 trace walk's chunk distribution (run under gpurun)
run() { env "$@" python bench.py --no-cpu-baseline --no-extra > gpurun_out/ab_tmp.json 2> gpurun_out/ab_tmp.err
python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_tmp.json').read().strip().splitlines()[-1])
print('$*', d['ms_per_step'], d['phase_us']['step1'])
"; }
run A=1
run A=2
run SLICECRAFT_B200_TRACE_SMMAJOR=1
run SLICECRAFT_B200_TRACE_STATIC=94
run SLICECRAFT_B200_TRACE_STATIC=97
run SLICECRAFT_B200_TRACE_STATIC=100
run SLICECRAFT_B200_TRACE_STATIC=97 SLICECRAFT_B200_TRACE_CHUNKS=512
run SLICECRAFT_B200_TRACE_STATIC=97 SLICECRAFT_B200_TRACE_CHUNKS=256
