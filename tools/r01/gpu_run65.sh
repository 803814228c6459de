# STN-GPe bifurcation: register cap of the throughput kernel (min blocks per SM) -- the 32-register
# build reloads two constant pairs with LDC every step (MIO queue, shared with MUFU).
for m in 16 12 10 8; do r=$(FF_TUNE_MINB_P2_T128=$m timeout 300 python bench.py --config stn_bif3d --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"); echo "stn_bif3d minb $m: $r"; done
for m in 16 12; do r=$(FF_TUNE_MINB_P2_T128=$m timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"); echo "lorenz minb $m: $r"; done
