# Lorenz, 4 particles per thread (long launches): RK4 unroll 1 / 2 / 4.
for u in 1 2 4; do for v in "" "--S 1000" "--S 10"; do r=$(FF_TUNE_UNROLL=$u timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'])"); echo "unroll $u [$v]: $r"; done; done
