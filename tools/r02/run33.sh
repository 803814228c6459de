# per-launch-length redraw variant (p4: per thread at >= 50 steps, cooperative below): reset + P3 suites, timings
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_reset.py tests/test_gpu_fullsize_p3.py tests/test_gpu_graph.py tests/test_gpu_exchange.py -m gpu -q -rf -x 2>&1 | tail -2
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for rep in 1 2; do
BARGS="--S 10" run s10 X=1
BARGS="--S 100" run s100 X=1
BARGS="--S 1 --no-image" run s1_noimage X=1
done
