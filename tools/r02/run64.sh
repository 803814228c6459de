# bench-table row for integration-only S = 1 frames after the image-sum fix
D=gpurun_out/r02/final3
mkdir -p $D/table
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python bench.py --S 1 --no-image --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $D/table/lorenz3d_S1_noimage.json 2>/dev/null; tail -c 900 $D/table/lorenz3d_S1_noimage.json
