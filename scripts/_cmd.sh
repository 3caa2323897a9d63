python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
BENCH_BACKEND=gloo BENCH_COMM=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -v Warning | tail -3 | cut -c1-700
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 | cut -c1-300
