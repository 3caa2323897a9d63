# scratch command file for gpurun
set -u
OUT=gpurun_out/${TAG:-r2i}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_shrink.py -q > $OUT/pytest_shrink.log 2>&1; echo "pytest shrink rc=$?"; tail -30 $OUT/pytest_shrink.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -8 $OUT/pytest.log
