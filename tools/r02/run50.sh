# FMA-bound small systems: 4 per thread for every launch length (5-7 steps included): suites + timings
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -2
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for S in 1 5 7 10 100; do BARGS="--S $S" run lz_s$S X=1; done
