# integration-only Lorenz frames (no reset, no image) at S = 10 / 100 / 1000: the per-tile and per-launch cost left at S = 100; with reset / image for the split
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
run() { tag=$1; shift; timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', '%.4e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']), 'frame %.1f us'%(1000*d['ms_per_step']))"; }
for S in 10 100 1000; do
  run bare_S$S --S $S --no-reset --no-image
  run reset_S$S --S $S --no-image
  run image_S$S --S $S --no-reset
  run both_S$S --S $S
done
run bare_S1 --S 1 --no-reset --no-image
run reset_S1 --S 1 --no-image
