# scratch command file for gpurun
set -u
OUT=gpurun_out/${TAG:-r2m}; mkdir -p $OUT
BMINRES_NVCC_EXTRA="-DK3B_PROF" python -c "from paper_1301_2102_b200 import _build; _build.build(force=True)" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
for p in 8 16 32; do K3B_PROF=1 timeout 300 python scripts/trace_k3b.py $p 20 2>&1 | tail -4; done
python -c "import __graft_entry__ as g; g.build()" > $OUT/build2.log 2>&1 || { echo BUILD FAIL; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
