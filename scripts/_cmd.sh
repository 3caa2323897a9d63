# scratch command file for gpurun
set -u
OUT=gpurun_out/${TAG:-r2d}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
CMD="python bench.py --config 4 --steps 1 --warmup 1 --iters 256 --no-kernel-timing --no-e2e --no-cpu-baseline --secondary none --time-to-tol none"
$CMD > $OUT/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1u_|k1_dmma|k2_dmma|k1a_" -s 12 -c 4 -o $OUT/full4 $CMD > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?"; tail -3 $OUT/ncu_full.log
