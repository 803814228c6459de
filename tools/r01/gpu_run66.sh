# Lorenz-class (dim <= 4) throughput kernel ff_step_p2_t128: register cap (min blocks per SM of 128
# threads: 16 -> 32 registers, 12 -> 40, 10 -> 48, 8 -> 64) over the Lorenz workloads, twice.
for rep in 1 2; do
for m in 16 14 12 10 8; do for v in "" "--S 10" "--S 1" "--S 1000" "--config sweep" "--config lorenz3d_collapsed"; do r=$(FF_TUNE_MINB_P2_T128=$m timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"); echo "minb $m [$v]: $r"; done; done
done
