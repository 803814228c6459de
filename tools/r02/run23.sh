# A/B/C on one box: reset redraw per thread (0), always warp-cooperative (1), cooperative when it needs fewer rounds (2)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for rep in 1 2; do
for m in 0 1 2; do
BARGS="--S 1" run s1_r$m FF_TUNE_REDRAW=$m
BARGS="--S 10" run s10_r$m FF_TUNE_REDRAW=$m
BARGS="--S 100" run s100_r$m FF_TUNE_REDRAW=$m
BARGS="--config stn_bif3d" run bif_r$m FF_TUNE_REDRAW=$m
done
done
