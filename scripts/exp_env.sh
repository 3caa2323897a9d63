#!/bin/bash
# Launch-shape experiments: one bench run per environment setting, phase times per block step.
# usage (via gpurun): bash scripts/exp_env.sh TAG CONFIG ITERS "ENV1" "ENV2" ...   ("" = defaults)
set -u
TAG=$1; CFG=$2; IT=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -f paper_1301_2102_b200/libbminres.so ] || python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 600 python bench.py --config $CFG --iters $IT --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
      --secondary none --time-to-tol none --precond none > $OUT/b$i.json 2> $OUT/b$i.err
  python - "$OUT/b$i.json" "$e" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as ex:
    print(sys.argv[2], "FAILED", ex); sys.exit()
r = d.get("roofline") or {}
ph = {k: round(v) for k, v in (r.get("phase_us_per_block_step") or {}).items()}
print(f"[{sys.argv[2]}] {d['value']:.0f} it/s  step_frac {d['step_roofline']['frac_of_measured']:.3f}  "
      f"clk {d.get('clocks',{}).get('sm_mhz')}  {ph}")
PY
done
