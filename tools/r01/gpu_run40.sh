# Register-operand microbenchmarks + Lorenz bench after the 3-register-FFMA2 penalty.
./tools/ubench/pipes 2>&1 | sed -n 6,11p
for v in "" "--S 1000" "--config hh"; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"; done
