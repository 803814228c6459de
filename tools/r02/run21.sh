# warp-cooperative reset redraw: reset + P3 + parity suites, then S = 1 / 10 / 100 and HH / bifurcation timings
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_reset.py tests/test_gpu_fullsize_p3.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -rf -x 2>&1 | tail -3
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'], d['roofline']['bound'], round(d['roofline']['frac'],3))"; }
BARGS="--S 1" run s1 X=1
BARGS="--S 10" run s10 X=1
BARGS="--S 100" run s100 X=1
BARGS="--config hh" run hh X=1
BARGS="--config stn_bif3d" run bif X=1
