# S = 1 frame with the round-2 kernel: pairs (default) vs 4 particles per thread (6 / 8 blocks/SM)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for rep in 1 2; do
BARGS="--S 1" run p2_m12 X=1
BARGS="--S 1 --ppt 4 --tpb 128" run p4_m6 X=1
BARGS="--S 1 --ppt 4 --tpb 128" run p4_m8 FF_TUNE_MINB_P4=8
BARGS="--S 1 --ppt 2 --tpb 256" run p2_t256 X=1
done
