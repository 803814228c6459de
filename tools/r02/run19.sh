# S = 10 frames: reset on / off, kernel variants
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'], d['roofline']['bound'], round(d['roofline']['frac'],3))"; }
BARGS="--S 10" run s10 X=1
BARGS="--S 10 --no-reset" run s10_noreset X=1
BARGS="--S 10 --no-image" run s10_noimage X=1
BARGS="--S 10 --ppt 2 --tpb 128" run s10_p2 X=1
BARGS="--S 10 --ppt 2 --tpb 256" run s10_p2_256 X=1
BARGS="--S 1" run s1 X=1
BARGS="--S 2" run s2 X=1
