# one-loop redraw (shared Philox for both modes): reset suite, then A/B/C on one box (0 per thread, 1 cooperative, 2 hybrid)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_reset.py tests/test_gpu_fullsize_p3.py -m gpu -q -rf -x 2>&1 | tail -2
FF_TUNE_REDRAW=0 timeout 900 python -m pytest tests/test_gpu_reset.py -m gpu -q -rf -x -k "density or lifted" 2>&1 | tail -1
FF_TUNE_REDRAW=1 timeout 900 python -m pytest tests/test_gpu_reset.py -m gpu -q -rf -x -k "density or lifted" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for rep in 1 2; do
for m in 0 1 2; do
BARGS="--S 10" run s10_r$m FF_TUNE_REDRAW=$m
BARGS="--S 100" run s100_r$m FF_TUNE_REDRAW=$m
BARGS="--config stn_bif3d" run bif_r$m FF_TUNE_REDRAW=$m
done
done
