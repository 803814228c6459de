# kernel choice in the gaps: Lorenz S = 5 / 7 (pairs by default) and STN-GPe bifurcation S = 4 / 10 / 30 (pairs by default for >= 5 steps)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for S in 5 7; do
BARGS="--S $S" run lz_s${S}_default X=1
BARGS="--S $S --ppt 4 --tpb 128" run lz_s${S}_p4 X=1
done
for S in 4 10 30; do
BARGS="--S $S --config stn_bif3d" run bif_s${S}_default X=1
BARGS="--S $S --config stn_bif3d --ppt 4 --tpb 128" run bif_s${S}_p4 X=1
BARGS="--S $S --config stn_bif3d --ppt 2 --tpb 128" run bif_s${S}_p2 X=1
done
