# e2e: callers x streams
mkdir -p gpurun_out/r2_52
for cs in "2 2" "2 3" "3 2" "4 1" "2 4"; do set -- $cs; timeout 900 python bench.py --no-cpu-baseline --steps 30 --e2e-callers $1 --e2e-streams $2 > gpurun_out/r2_52/b_$1_$2.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/r2_52/b_$1_$2.json'));print('callers $1 streams $2', round(d['value']), round(d['e2e']['value']), round(d['e2e'].get('single_caller_value',0)))"; done
