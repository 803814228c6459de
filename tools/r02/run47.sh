# long launches re-check with the round-2 kernel: STN-GPe bifurcation and sweep across kernel variants
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 4 --no-cpu-baseline --no-e2e $BARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.3e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; }
for rep in 1 2; do
BARGS="--config stn_bif3d" run bif_default X=1
BARGS="--config stn_bif3d --ppt 4 --tpb 128" run bif_p4 X=1
BARGS="--config stn_bif3d --ppt 2 --tpb 128" run bif_p2_128 X=1
BARGS="--config sweep" run sweep_default X=1
BARGS="--config sweep --ppt 2 --tpb 256" run sweep_p2_256 X=1
done
