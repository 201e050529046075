# e2e: more callers at one stream each
mkdir -p gpurun_out/r2_53
for cs in "3 1" "4 1" "6 1" "8 1" "4 2"; do set -- $cs; timeout 900 python bench.py --no-cpu-baseline --steps 32 --e2e-callers $1 --e2e-streams $2 > gpurun_out/r2_53/b_$1_$2.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/r2_53/b_$1_$2.json'));print('callers $1 streams $2', round(d['value']), round(d['e2e']['value']), round(d['e2e'].get('single_caller_value',0)))"; done
