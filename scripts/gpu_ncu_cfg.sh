#!/bin/bash
# ncu --set full of one config's step kernels + its launch list (as gpu_check.sh does for configs 4 and 2).
# usage (via gpurun): bash scripts/gpu_ncu_cfg.sh TAG CONFIG [SKIP] [COUNT]
set -u
TAG=$1; CFG=$2; SKIP=${3:-40}; CNT=${4:-12}
OUT=gpurun_out/$TAG; mkdir -p $OUT; R=/tmp/ncu_$TAG; mkdir -p $R
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; exit 1; }
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --iters 400 --no-kernel-timing --no-e2e --no-cpu-baseline --secondary none --time-to-tol none --precond none"
$CMD > $OUT/plain_cfg$CFG.log 2>&1 || { echo PLAIN FAIL; tail -5 $OUT/plain_cfg$CFG.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_cfg$CFG.csv $CMD > $OUT/ncu_launch_cfg$CFG.log 2>&1; echo "ncu-launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k1_|k1u_|k1a_|k2_|k3b_|k_reduce|k_red2f" -s $SKIP -c $CNT \
  -o $R/full_cfg$CFG $CMD > $OUT/ncu_full_cfg$CFG.log 2>&1; echo "ncu-full rc=$?"
python profiles/summarize_ncu.py --rep $R/full_cfg$CFG.ncu-rep > $OUT/full_cfg${CFG}_summary.md 2>&1
ncu -i $R/full_cfg$CFG.ncu-rep --page raw --csv > $OUT/full_cfg${CFG}_raw.csv 2>/dev/null
ls -la $OUT
