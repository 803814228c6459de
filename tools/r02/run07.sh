# reset redraw loop: rolled vs unrolled over the thread's particles (S = 100 and S = 1, Lorenz with reset)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'])"; }
for i in 1 2; do
BARGS="--S 100" run s100 X=1
BARGS="--S 100" run s100_unroll FF_TUNE_RESET_UNROLL=1
BARGS="--S 100 --no-reset" run s100_noreset X=1
done
BARGS="--S 1" run s1 X=1
BARGS="--S 1" run s1_unroll FF_TUNE_RESET_UNROLL=1
