# device-resident measurement with concurrent callers
mkdir -p gpurun_out/r2_56
for c in C3 C1 C2 C4; do for k in "1 3" "4 1" "8 1" "4 2"; do set -- $k; timeout 600 python bench.py --config $c --no-cpu-baseline --callers $1 --caller-streams $2 > gpurun_out/r2_56/b_${c}_$1_$2.json 2> gpurun_out/r2_56/b_${c}_$1_$2.err; python -c "
import json;d=json.load(open('gpurun_out/r2_56/b_${c}_$1_$2.json'));print('$c callers $1 x $2', round(d['value']), 'e2e', round(d['e2e']['value']), 'launches', d['gpu_launches'], d['status_ok'] if 'status_ok' in d else '')" || tail -3 gpurun_out/r2_56/b_${c}_$1_$2.err; done; done
