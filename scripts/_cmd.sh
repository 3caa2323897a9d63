# scratch command file for gpurun
set -u
OUT=gpurun_out/${TAG:-r2h}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
for p in 8 16 32; do timeout 300 python scripts/trace_k3b.py $p 2>&1 | tail -2; done
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $OUT/pytest.log
for extra in "--config 3" "--config 2"; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --secondary none --time-to-tol none --steps 5 $extra > $OUT/bench.json 2> $OUT/bench.err; echo "bench $extra rc=$?"
  python - <<PY
import json
d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print('value %.0f it/s  ms/step %.3f  step_frac %.3f clocks %s launches %s' % (d['value'], d['ms_per_step'], d['step_roofline']['frac_of_measured'], d['clocks'], d['gpu_launches']))
print('phases', {k: round(v,1) for k,v in (r.get('phase_us_per_block_step') or {}).items()})
PY
done
