# HH ring pipe-balance knobs with the round-2 kernel: sigmoid pairs off, exponentials moved to the FMA pipe
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
BARGS="--config hh"
run default X=1
run nopairs FF_TUNE_RCP_PAIRS=0
run exp4 FF_TUNE_EXP2P_STEP=4
run rcpp1 FF_TUNE_RCPP_STAGES=1
run default2 X=1
