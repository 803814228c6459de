# Measurement only (not a product change): the 3-D projection with rcp*mul instead of the exact
# IEEE division, S = 100 and S = 10 with and without the image (the division is not the cost).
for i in 1 2; do for v in "" "--no-image" "--S 10" "--S 10 --no-image"; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.1f us'%(1000*d['kernel_ms_mean']))"; done; done
