# pass A with interleaved bisections (A/B vs r2_54) + device-resident streams per config
mkdir -p gpurun_out/r2_55
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_55/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_55/pytest.log
for c in "C3 296" "C4 512"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_55/ab.log
for c in C1 C2 C4; do for s in 3 6 8; do timeout 600 python bench.py --config $c --no-cpu-baseline --e2e-callers 1 --streams $s > gpurun_out/r2_55/b_${c}_$s.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/r2_55/b_${c}_$s.json'));print('$c streams $s', round(d['value']), round(d['e2e']['value']))"; done; done
