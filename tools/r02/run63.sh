# short launches with static tiles + TMA prefetch of the next two tiles (FF_TUNE_PREFETCH=1): parity suites with it on, then S = 1 / 2 / 4 A/B
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
FF_TUNE_PREFETCH=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reset.py tests/test_gpu_fullsize_p3.py tests/test_gpu_graph.py tests/test_gpu_exchange.py tests/test_gpu_exchange_push.py -m gpu -q -k "not 1B" 2>&1 | tail -3
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.4e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), 'frame %.1f us'%(1000*d['ms_per_step']))"; }
for i in 1 2; do
for S in 1 2 4; do
BARGS="--S $S --no-image" run noimg_S${S}_base FF_TUNE_PREFETCH=0
BARGS="--S $S --no-image" run noimg_S${S}_pf FF_TUNE_PREFETCH=1
BARGS="--S $S" run img_S${S}_base FF_TUNE_PREFETCH=0
BARGS="--S $S" run img_S${S}_pf FF_TUNE_PREFETCH=1
done
BARGS="--S 1 --config stn_bif3d" run bif_S1_base FF_TUNE_PREFETCH=0
BARGS="--S 1 --config stn_bif3d" run bif_S1_pf FF_TUNE_PREFETCH=1
BARGS="--S 1 --config sweep" run sweep_S1_base FF_TUNE_PREFETCH=0
BARGS="--S 1 --config sweep" run sweep_S1_pf FF_TUNE_PREFETCH=1
done
