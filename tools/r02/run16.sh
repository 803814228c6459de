# S = 100 frame cost split: reset on/off x image on/off; RK4 unroll of the p4 kernel
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'])"; }
BARGS="--S 100" run reset_image X=1
BARGS="--S 100 --no-reset" run noreset_image X=1
BARGS="--S 100 --no-image" run reset_noimage X=1
BARGS="--S 100 --no-image --no-reset" run noreset_noimage X=1
BARGS="--S 100" run reset_image_u4 FF_TUNE_UNROLL=4
BARGS="--S 100" run reset_image_u1 FF_TUNE_UNROLL=1
BARGS="--S 1000" run reset_image_s1000 X=1
