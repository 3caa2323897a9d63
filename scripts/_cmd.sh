bash scripts/gpu_quick.sh q14 ""
B="python bench.py --no-cpu-baseline --no-e2e --no-kernel-timing"
v() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value']), round(d['ms_per_step'],3))"; }
BMINRES_GRAPH_BLOCKS=1 $B | v gb1
BMINRES_GRAPH_BLOCKS=3 $B | v gb3
BMINRES_GRAPH_BLOCKS=6 $B | v gb6
