run() { env "$@" python bench.py --no-cpu-baseline --no-extra > gpurun_out/ab_tmp.json 2> gpurun_out/ab_tmp.err
python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_tmp.json').read().strip().splitlines()[-1])
print('$*', d['ms_per_step'], d['phase_us']['step1'], d['phase_us']['step2'])
"; }
run A=1
run SLICECRAFT_B200_SPLIT2=8
run SLICECRAFT_B200_SPLIT2=32
run SLICECRAFT_B200_SPLIT2=64
run SLICECRAFT_B200_SPLIT2=32 SLICECRAFT_B200_SPLIT_DEPTH2=2
run SLICECRAFT_B200_FILTER=0
