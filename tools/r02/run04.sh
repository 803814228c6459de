# S = 1 frame kernel experiments: all-static tiles, register prefetch of the next tile, register budget, 2 vs 4 particles/thread
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --S 1 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'])"; }
run base X=1
run static FF_TUNE_STATIC_ALL=2
run static_pf_m16 FF_TUNE_STATIC_ALL=2 FF_TUNE_PREFETCH=1
run static_pf_m12 FF_TUNE_STATIC_ALL=2 FF_TUNE_PREFETCH=1 FF_TUNE_MINB_P2_T128=12
run static_pf_m10 FF_TUNE_STATIC_ALL=2 FF_TUNE_PREFETCH=1 FF_TUNE_MINB_P2_T128=10
run static_m12 FF_TUNE_STATIC_ALL=2 FF_TUNE_MINB_P2_T128=12
BARGS="--ppt 4 --tpb 128"
run p4_base X=1
run p4_static FF_TUNE_STATIC_ALL=2
run p4_static_pf FF_TUNE_STATIC_ALL=2 FF_TUNE_PREFETCH=1
run p4_static_pf_m4 FF_TUNE_STATIC_ALL=2 FF_TUNE_PREFETCH=1 FF_TUNE_MINB_P4=4
BARGS="--no-image"
run noimg_base X=1
run noimg_static FF_TUNE_STATIC_ALL=2
run noimg_static_pf FF_TUNE_STATIC_ALL=2 FF_TUNE_PREFETCH=1
