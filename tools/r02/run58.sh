# HH ring register budget re-measured (NVRTC now fits 3 blocks/SM in 168 registers without spills): MINB 2 / 3 / 4, unroll 1 / 2
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config hh --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.4e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for i in 1 2; do
run m2 FF_TUNE_MINB_P2_T128=2
run m3 FF_TUNE_MINB_P2_T128=3
run m4 FF_TUNE_MINB_P2_T128=4
run m3_u1 FF_TUNE_MINB_P2_T128=3 FF_TUNE_UNROLL=1
run m3_u3 FF_TUNE_MINB_P2_T128=3 FF_TUNE_UNROLL=3
done
