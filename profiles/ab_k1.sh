# A/B of K1: direct 128-bit loads vs TMA-staged tiles (run under gpurun)
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --no-extra > gpurun_out/k1_tmp.json 2> gpurun_out/k1_tmp.err
python -c "
import json
d=json.loads(open('gpurun_out/k1_tmp.json').read().strip().splitlines()[-1])
r=d['roofline_texture']
print('$*', 'step', round(d['ms_per_step'],4), 'alone_us', r['launch_us'], r['frac'], 'pipeline_us', r['in_pipeline']['launch_us'], r['in_pipeline']['frac'], 'e2e', round(d['e2e']['ms_per_step'],3), d['phase_us']['tables_k2k3'], d['phase_us']['time_tables_main'])
"; }
for i in 1 2 3; do
run SLICECRAFT_B200_K1=ldg
run SLICECRAFT_B200_K1=tma SLICECRAFT_B200_K1_CTAS=3
run SLICECRAFT_B200_K1=tma SLICECRAFT_B200_K1_CTAS=2
done
