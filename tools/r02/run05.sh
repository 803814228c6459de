# shared-reciprocal projection + identity-axes fast path: division check, parity, S=1 / S=100 timings
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_division.py tests/test_gpu_parity.py tests/test_gpu_reset.py -m gpu -q -rf -x 2>&1 | tail -5
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'])"; }
BARGS="--S 1" run s1 X=1
BARGS="--S 1 --no-reset" run s1_noreset X=1
BARGS="--S 1 --no-image" run s1_noimg X=1
BARGS="--S 1 --no-image --no-reset" run s1_noimg_noreset X=1
BARGS="--S 100" run s100 X=1
BARGS="--S 100 --no-reset" run s100_noreset X=1
