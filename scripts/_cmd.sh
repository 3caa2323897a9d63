python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/c45b
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
v() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(d['value']), round(d['ms_per_step'],2), 'K1', round(r['mean_launch_us']), round(r['frac'],3), {k: round(v) for k,v in r['phase_us_per_block_step'].items()})"; }
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 --iters 1024 --no-cpu-baseline --no-e2e | tee gpurun_out/c45b/cfg4.json | v cfg4
timeout 900 python bench.py --config 5 --steps 3 --warmup 1 --iters 1024 --no-cpu-baseline --no-e2e | tee gpurun_out/c45b/cfg5.json | v cfg5
timeout 900 python bench.py --no-cpu-baseline --no-e2e | v cfg2
