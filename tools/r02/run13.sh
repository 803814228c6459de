# RED / streaming overlap microbenchmark; short-launch register budget (12 vs 16 blocks/SM) at S = 1, 2, 4
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/red_stream tools/ubench/red_stream.cu && /tmp/red_stream | tee gpurun_out/r02/ubench_red_stream.txt
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), d['image_sum_last_frame'])"; }
for S in 1 2 4 7; do
BARGS="--S $S" run s${S}_m16 X=1
BARGS="--S $S" run s${S}_m12 FF_TUNE_MINB_P2_T128=12
BARGS="--S $S" run s${S}_m10 FF_TUNE_MINB_P2_T128=10
done
BARGS="--S 1 --no-reset" run s1_m12_noreset FF_TUNE_MINB_P2_T128=12
