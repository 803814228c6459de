mkdir -p gpurun_out/table
for c in lorenz3d hh sweep stn stn_bif3d lorenz3d_collapsed lorenz1b; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-e2e > gpurun_out/table/$c.json 2>/dev/null; done
for s in 1 10 1000; do timeout 300 python bench.py --config lorenz3d --S $s --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/table/lorenz3d_S$s.json 2>/dev/null; done
timeout 300 python bench.py --config lorenz3d --S 1 --no-image --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/table/lorenz3d_S1_noimage.json 2>/dev/null
ls -la gpurun_out/table
