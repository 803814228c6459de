# SURVEY 8(d) histogram-regime benchmark: projection + histogram cost as a fraction of the launch,
# S in {1, 100}, dispersed (r = 28) vs collapsed (r = 0.5 after 4000 steps: every particle in ~1 pixel).
for c in lorenz3d lorenz3d_collapsed; do for S in 1 100; do for img in "" "--no-image"; do
timeout 300 python bench.py --config $c --S $S --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $img 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c S=$S ${img:-image}', '%.4g'%d['value'], '%.2f us'%(1000*d['kernel_ms_mean']))"
done; done; done
