#!/bin/bash
# One GPU round trip: parity tests, bench, ncu launch list, ncu --set full of the step kernels.
# usage (via gpurun): bash scripts/gpu_check.sh TAG [tests|notests] [full|nofull]
set -u
TAG=${1:-run}; TESTS=${2:-tests}; FULL=${3:-full}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
if [ "$TESTS" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
fi
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 600 $OUT/bench.json
CMD="python bench.py --steps 1 --warmup 1 --iters 400 --no-kernel-timing --no-e2e --no-cpu-baseline --secondary none --time-to-tol none --precond none"
$CMD > $OUT/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
if [ "$FULL" = full ]; then
  # reports go to /tmp (gpurun copies back at most 64 MiB); summaries + raw csv into $OUT
  R=/tmp/ncu_$TAG; mkdir -p $R
  # config 4's step kernels (skip the start block and the first block steps), then config 2's
  CMD2="python bench.py --steps 1 --warmup 1 --iters 800 --no-kernel-timing --no-e2e --no-cpu-baseline --secondary none --time-to-tol none --precond none"
  $CMD2 > $OUT/plain2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k1_|k1u_|k1a_|k2_|k3b_|k_reduce" -s 40 -c 12 \
    -o $R/full $CMD2 > $OUT/ncu_full.log 2>&1; echo "ncu-full rc=$?"
  CMD3="python bench.py --config 2 --steps 1 --warmup 1 --iters 400 --no-kernel-timing --no-e2e --no-cpu-baseline --secondary none --time-to-tol none --precond none"
  $CMD3 > $OUT/plain3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_cfg2.csv $CMD3 > $OUT/ncu_launch3.log 2>&1; echo "ncu-launch-cfg2 rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_|k2_|k3b_|k_reduce|k_red2f" -s 100 -c 10 \
    -o $R/full_cfg2 $CMD3 > $OUT/ncu_full3.log 2>&1; echo "ncu-full-cfg2 rc=$?"
  for r in full full_cfg2; do
    [ -f $R/$r.ncu-rep ] || continue
    python profiles/summarize_ncu.py --rep $R/$r.ncu-rep > $OUT/${r}_summary.md 2>&1
    ncu -i $R/$r.ncu-rep --page raw --csv > $OUT/${r}_raw.csv 2>/dev/null
    [ $(stat -c %s $R/$r.ncu-rep) -lt 20000000 ] && cp $R/$r.ncu-rep $OUT/
  done
  ls -la $OUT
fi
