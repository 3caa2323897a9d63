#!/bin/bash
# Compile-time + environment experiments: for each "DEFINES|ENV" spec, rebuild with
# BMINRES_NVCC_EXTRA=DEFINES, then one bench run with ENV (phase times per launch).
# usage (via gpurun): bash scripts/exp_build.sh TAG CONFIG ITERS "DEFS|ENV" ...
set -u
TAG=$1; CFG=$2; IT=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in "$@"; do
  defs="${spec%%|*}"; envs="${spec#*|}"
  BMINRES_NVCC_EXTRA="$defs" python -c "from paper_1301_2102_b200 import _build; _build.build(force=True)" > $OUT/build.log 2>&1 || { echo "[$spec] BUILD FAIL"; tail -5 $OUT/build.log; continue; }
  env $envs timeout 600 python bench.py --config $CFG --iters $IT --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
      --secondary none --time-to-tol none --precond none > $OUT/b.json 2> $OUT/b.err
  python - "$OUT/b.json" "$spec" <<'PY'
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
python -c "from paper_1301_2102_b200 import _build; _build.build(force=True)" > $OUT/build.log 2>&1
