# ncu source-level capture of the S = 10 frame with reset (why binning the backward group costs ~38 us)
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 8 -c 1 -o gpurun_out/r02/s10_full python bench.py --S 10 --steps 1 --warmup 8 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 8 -c 1 -o gpurun_out/r02/s10_noreset_full python bench.py --S 10 --steps 1 --warmup 8 --no-cpu-baseline --no-e2e --no-reset > /dev/null 2>&1; echo "rc=$?"
