# short launches (S = 1, 2, 4; with / without image): pairs vs 4 per thread at 6 / 8 blocks/SM; STN-GPe bifurcation at S = 1
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for S in 1 2 4; do
BARGS="--S $S --ppt 2 --tpb 128" run img_s${S}_p2 X=1
BARGS="--S $S --ppt 4 --tpb 128" run img_s${S}_p4m6 X=1
BARGS="--S $S --ppt 4 --tpb 128" run img_s${S}_p4m8 FF_TUNE_MINB_P4=8
BARGS="--S $S --no-image --ppt 4 --tpb 128" run noimg_s${S}_p4m6 X=1
BARGS="--S $S --no-image --ppt 4 --tpb 128" run noimg_s${S}_p4m8 FF_TUNE_MINB_P4=8
done
BARGS="--S 1 --config stn_bif3d --ppt 2 --tpb 128" run bif_s1_p2 X=1
BARGS="--S 1 --config stn_bif3d --ppt 4 --tpb 128" run bif_s1_p4m6 X=1
BARGS="--S 1 --config stn_bif3d --ppt 4 --tpb 128" run bif_s1_p4m8 FF_TUNE_MINB_P4=8
BARGS="--S 1 --config stn_bif3d" run bif_s1_default X=1
