# histogram warp regime judged on the first lane holding a particle: histogram / render / P3 tests, S=1 and S=100 timings
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render.py tests/test_gpu_fullsize_p3.py -m gpu -q -rf -x 2>&1 | tail -3
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'])"; }
BARGS="--S 1" run s1 X=1
BARGS="--S 100" run s100 X=1
BARGS="--S 1 --config lorenz3d_collapsed" run collapsed_s1 X=1
BARGS="--S 100 --config lorenz3d_collapsed" run collapsed_s100 X=1
