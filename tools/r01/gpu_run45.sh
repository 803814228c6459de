# Per-launch fixed cost of the Lorenz frame: S sweep with and without the image.
for S in 20 50 100 200 400; do for img in "" "--no-image"; do timeout 300 python bench.py --S $S --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $img 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S=$S $img', '%.4g'%d['value'], '%.1f us'%(1000*d['kernel_ms_mean']))"; done; done
