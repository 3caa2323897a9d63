# scratch command file for gpurun
set -u
OUT=gpurun_out/${TAG:-r2m}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "warp_specialised or split_mode or deferred or full_size_config_first" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest.log
for extra in "--config 4" "--config 5"; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --secondary none --time-to-tol none --steps 5 $extra > $OUT/bench.json 2> $OUT/bench.err; echo "bench $extra rc=$?"
  python - <<PY
import json
d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print('value %.0f it/s  ms/step %.3f  step_frac %.3f clocks %s launches %s' % (d['value'], d['ms_per_step'], d['step_roofline']['frac_of_measured'], d['clocks'], d['gpu_launches']))
print('phases', {k: round(v,1) for k,v in (r.get('phase_us_per_block_step') or {}).items()})
PY
done
