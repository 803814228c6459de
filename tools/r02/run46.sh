# short launches now 4 per thread at 8 blocks/SM (image or not): parity suites, then S = 1 / 2 / 4 / 100 timings
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -3
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['roofline']['bound'], round(d['roofline']['frac'],3))"; }
for rep in 1 2; do
BARGS="--S 1" run s1 X=1
BARGS="--S 1 --no-image" run s1_noimg X=1
BARGS="--S 2" run s2 X=1
BARGS="--S 4" run s4 X=1
BARGS="--S 100" run s100 X=1
done
