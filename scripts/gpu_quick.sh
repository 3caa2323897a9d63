#!/bin/bash
# Quick GPU iteration: build, parity tests, bench (no CPU baseline).  usage: bash scripts/gpu_quick.sh TAG [extra bench args]
set -u
TAG=${1:-q}; shift || true
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for extra in "$@"; do
  echo "== bench $extra"
  eval timeout 600 python bench.py --no-cpu-baseline --no-e2e $extra > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
  python -c "
import json,sys
d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print('value %.0f it/s  ms/step %.3f  step_frac %.3f' % (d['value'], d['ms_per_step'], d['step_roofline']['frac_of_measured']))
print('phases', {k: round(v,1) for k,v in (r.get('phase_us_per_block_step') or {}).items()})
" 2>&1 || tail -20 $OUT/bench.err
done
