# Confirm the unroll factor (long-launch build): Lorenz workloads and the STN-GPe bifurcation, twice.
for rep in 1 2; do
for u in 2 3 4; do for v in "" "--S 10" "--S 1000" "--config sweep"; do r=$(FF_TUNE_UNROLL=$u timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"); echo "unroll $u [$v]: $r"; done; done
for u in 4 8; do r=$(FF_TUNE_UNROLL=$u timeout 300 python bench.py --config stn_bif3d --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"); echo "stn_bif3d unroll $u: $r"; done
done
