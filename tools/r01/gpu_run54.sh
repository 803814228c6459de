# HH ring: blocks per SM of the packed 128-thread kernel (register budget vs occupancy).
for m in 2 3 4; do r=$(FF_TUNE_MINB_P2_T128=$m timeout 300 python bench.py --config hh --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"); echo "hh minb $m: $r"; done
