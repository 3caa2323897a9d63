run() { echo -n "$1: "; env $1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-kernel-timing 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']))"; }
for r in 1 2; do run X=0; run BMINRES_NO_XDEFER=1; run BMINRES_NO_RED2F=1; run BMINRES_NO_EARLY_RED2=1; run BMINRES_NO_ROWK=1; done
