# e2e with concurrent callers
mkdir -p gpurun_out/r2_49
for c in 1 2 3; do timeout 900 python bench.py --no-cpu-baseline --e2e-callers $c > gpurun_out/r2_49/bench_c$c.json 2> gpurun_out/r2_49/bench_c$c.err; echo "callers $c rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/r2_49/bench_c$c.json'));print(d['value'], d['e2e'])"; done
