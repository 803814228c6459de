# HH ring register budget again (the packed kernel now allocates 220 registers at 2 blocks/SM)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
BARGS="--config hh"
run hh_m2 X=1
run hh_m3 FF_TUNE_MINB_P2_T128=3
run hh_m2_u2 FF_TUNE_UNROLL=2
BARGS="--config hh --ppt 2 --tpb 256"
run hh_t256 X=1
