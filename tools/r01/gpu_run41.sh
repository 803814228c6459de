# Round-1 evidence refresh: smoke, GPU tests, bench table over every workload, default bench line,
# launch list of the default bench command, ncu --set full captures of the top kernels.
mkdir -p gpurun_out/table gpurun_out/ncu
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/r01_bench_default.json 2> gpurun_out/r01_bench_default.err; tail -c 300 gpurun_out/r01_bench_default.json; echo
for c in lorenz3d hh sweep stn stn_bif3d lorenz3d_collapsed lorenz1b; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/table/$c.json 2>/dev/null; done
for s in 1 10 1000; do timeout 300 python bench.py --config lorenz3d --S $s --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/table/lorenz3d_S$s.json 2>/dev/null; done
timeout 300 python bench.py --config lorenz3d --S 1 --no-image --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/table/lorenz3d_S1_noimage.json 2>/dev/null
timeout 300 python bench.py --config lorenz3d --exchange fused --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/table/lorenz3d_exchange_fused.json 2>/dev/null
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01_bench_reference.json 2>/dev/null; tail -c 300 gpurun_out/r01_bench_reference.json; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for spec in "lorenz3d_S100:" "lorenz3d_S1:--S 1" "lorenz3d_S1_noimage:--S 1 --no-image" "hh_S100:--config hh" "sweep_S100:--config sweep" "stn_bif3d_S100:--config stn_bif3d"; do
  name=${spec%%:*}; args=${spec#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/ncu/$name python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $args > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_exchange -s 3 -c 1 -o gpurun_out/ncu/exchange_w1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --exchange fused > /dev/null 2>&1
ls gpurun_out/ncu gpurun_out/table
