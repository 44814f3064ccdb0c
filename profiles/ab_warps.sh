# A/B of the step-1 trace walk's chunk distribution (run under gpurun)
run() { env "$@" python bench.py --no-cpu-baseline --no-extra > gpurun_out/ab_tmp.json 2> gpurun_out/ab_tmp.err
python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_tmp.json').read().strip().splitlines()[-1])
print('$*', d['ms_per_step'], d['phase_us']['step1'])
"; }
run SLICECRAFT_B200_TRACE_STATIC=88
run SLICECRAFT_B200_TRACE_STATIC=80
run SLICECRAFT_B200_TRACE_STATIC=75
run SLICECRAFT_B200_TRACE_STATIC=70
run SLICECRAFT_B200_TRACE_STATIC=60
run SLICECRAFT_B200_TRACE_STATIC=50
run SLICECRAFT_B200_TRACE_STATIC=80
run SLICECRAFT_B200_TRACE_STATIC=70
