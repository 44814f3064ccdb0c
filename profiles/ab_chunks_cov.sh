# covering family, lambda 0.3: trace chunk size A/B (run under gpurun)
run() { env "$@" python bench.py --no-cpu-baseline --no-extra --lambda 0.3 --coverage 1 > gpurun_out/abc_tmp.json 2> gpurun_out/abc_tmp.err
python -c "
import json,sys
d=json.loads(open('gpurun_out/abc_tmp.json').read().strip().splitlines()[-1])
print('$*', d['ms_per_step'], d['phase_us']['step1'], d['phase_us']['step2'])
"; }
run A=1
run SLICECRAFT_B200_TRACE_CHUNKS=512
run SLICECRAFT_B200_TRACE_CHUNKS=256
run SLICECRAFT_B200_TRACE_CHUNKS=128
run SLICECRAFT_B200_TRACE_CHUNKS=64
