# STN-GPe bifurcation pipe balance re-check with the round-2 kernel: exponentials on the FMA pipe per particle-step (K) and pair-reciprocal stages (R)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
BARGS="--config stn_bif3d"
run default X=1
for R in 0 2; do run R$R FF_TUNE_RCPP_STAGES=$R; done
for K in 1 2; do run K$K FF_TUNE_EXP2P_STEP=$K; done
run nopairs FF_TUNE_RCP_PAIRS=0
run default2 X=1
