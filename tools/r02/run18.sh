# round-2 bench table: every workload with the default launch (and S = 1 / 10 / 1000 / no-image variants of lorenz3d)
mkdir -p gpurun_out/r02/table
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for c in lorenz3d stn hh sweep stn_bif3d lorenz3d_collapsed; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/r02/table/$c.json 2>/dev/null; echo "$c $?"
done
timeout 600 python bench.py --config lorenz1b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/table/lorenz1b.json 2>/dev/null; echo "lorenz1b $?"
for S in 1 10 1000; do timeout 300 python bench.py --S $S --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/table/lorenz3d_S$S.json 2>/dev/null; done
timeout 300 python bench.py --S 1 --no-image --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/table/lorenz3d_S1_noimage.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02/table_reference.json 2>/dev/null
python tools/bench_table.py gpurun_out/r02/table gpurun_out/r02/bench_table.md > /dev/null; cat gpurun_out/r02/bench_table.md
