# scratch command file for gpurun
set -u
OUT=gpurun_out/${TAG:-r2g}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
for p in 8 16 32; do timeout 300 python scripts/trace_k3b.py $p 2>&1 | tail -2; done
timeout 600 python -m pytest tests/test_studies.py -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
mkdir -p $OUT/prof
timeout 1500 python scripts/study_block_vs_seq.py --N 200 --pairs 10 --out $OUT/prof/r02_study_block_vs_seq.json > $OUT/study.log 2>&1; echo "study rc=$?"; tail -30 $OUT/study.log
