# more callers?
mkdir -p gpurun_out/r2_65
for k in "8 8" "12 12" "16 16"; do set -- $k; timeout 900 python bench.py --no-cpu-baseline --steps 48 --callers $1 --e2e-callers $2 > gpurun_out/r2_65/b_$1.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/r2_65/b_$1.json'));print('callers $1', round(d['value']), 'e2e', round(d['e2e']['value']))"; done
