timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
run() { echo -n "$1 $2: "; env $1 timeout 600 python bench.py $2 --no-e2e --no-cpu-baseline --no-kernel-timing 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']))"; }
run X=0 "--steps 10 --warmup 3"
run X=0 "--config 3 --steps 5 --warmup 3"
run BMINRES_NO_EARLY_RED1=1 "--config 3 --steps 5 --warmup 3"
