# A/B of step-1 walk source variants built as separate libraries (run under gpurun)
run() { env "$@" python bench.py --no-cpu-baseline --no-extra > gpurun_out/ab_tmp.json 2> gpurun_out/ab_tmp.err
python -c "
import json,sys
d=json.loads(open('gpurun_out/ab_tmp.json').read().strip().splitlines()[-1])
print('$*', d['ms_per_step'], d['phase_us']['step1'])
"; }
for i in 1 2; do
run A=base
for v in paper_2012_14792_b200/libvariant_*.so; do run SLICECRAFT_B200_LIB=$PWD/$v; done
done
