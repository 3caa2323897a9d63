bash scripts/gpu_quick.sh q12 ""
timeout 300 python scripts/trace_timeline.py 2 40 800
