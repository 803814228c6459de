# HH ring: the vtrap series under a warp-uniform branch (FF_TUNE_VTRAP_BRANCH) vs the branch-free select; parity with the knob on
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config hh --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.4e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for i in 1 2; do
run hh_select FF_TUNE_VTRAP_BRANCH=0
run hh_branch FF_TUNE_VTRAP_BRANCH=1
done
BARGS="--S 1000" run hh_select_S1000 FF_TUNE_VTRAP_BRANCH=0
BARGS="--S 1000" run hh_branch_S1000 FF_TUNE_VTRAP_BRANCH=1
FF_TUNE_VTRAP_BRANCH=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_frontend.py -m gpu -q -k "hh or vtrap or funcs or builtin or config3" 2>&1 | tail -3
