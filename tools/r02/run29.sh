# HH ring: RK4 unroll 1 vs 2 (A/B twice on one box); CUDA-graph frame capture tests
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
BARGS="--config hh"
for rep in 1 2; do run hh_u1 FF_TUNE_UNROLL=1; run hh_u2 FF_TUNE_UNROLL=2; run hh_u3 FF_TUNE_UNROLL=3; done
timeout 900 python -m pytest tests/test_gpu_graph.py -m gpu -q -rf 2>&1 | tail -3
