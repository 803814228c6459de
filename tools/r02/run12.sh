# packed (FMUL2/FFMA2) 3-D binning of particle pairs: parity first, then S=1 / S=100 timings and variants
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize_p3.py tests/test_gpu_parity.py -k "histogram or fused or p3 or bench_frame" -m gpu -q -rf -x 2>&1 | tail -4
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'])"; }
BARGS="--S 1"
run s1_packed X=1
run s1_scalar FF_TUNE_PACKED_BIN=0
run s1_packed_m12 FF_TUNE_MINB_P2_T128=12
run s1_packed_static FF_TUNE_STATIC_ALL=2
BARGS="--S 1 --ppt 4 --tpb 128"
run s1_p4_packed X=1
run s1_p4_packed_m8 FF_TUNE_MINB_P4=8
BARGS="--S 100"
run s100_packed X=1
run s100_scalar FF_TUNE_PACKED_BIN=0
BARGS="--S 10"
run s10_packed X=1
run s10_scalar FF_TUNE_PACKED_BIN=0
