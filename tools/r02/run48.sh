# round-2 evidence refresh after the short-launch change (4 per thread at 8 blocks/SM): suite, sanitizers, ncu, launch list, bench table, default + reference lines
# and the other kernels, launch list of the default command, bench table over every workload, default bench line
mkdir -p gpurun_out/r02/final2/table
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/r02/final2/pytest_gpu.log 2>&1; tail -3 gpurun_out/r02/final2/pytest_gpu.log
SAN="tests/test_gpu_parity.py::test_histogram_aggregation_regimes_exact tests/test_gpu_parity.py::test_histogram_warp_regime_with_dropped_leading_lanes tests/test_gpu_reset.py::test_redraws_bit_exact_at_any_reset_density tests/test_gpu_render.py"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $SAN -m gpu -q -p no:cacheprovider > gpurun_out/r02/final2/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -2 gpurun_out/r02/final2/sanitizer_memcheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest $SAN -m gpu -q -p no:cacheprovider > gpurun_out/r02/final2/sanitizer_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -2 gpurun_out/r02/final2/sanitizer_synccheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python -m pytest $SAN -m gpu -q -p no:cacheprovider > gpurun_out/r02/final2/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/r02/final2/sanitizer_racecheck.log
cap() { name=$1; shift; timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 4 -c 1 -o gpurun_out/r02/final2/$name python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e "$@" > /dev/null 2>&1; echo "$name $?"; }
cap lorenz3d_S100
cap lorenz3d_S1 --S 1
cap hh_S100 --config hh
cap stn_bif3d_S100 --config stn_bif3d
cap sweep_S100 --config sweep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/final2/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launch list $?"
for c in lorenz3d stn hh sweep stn_bif3d lorenz3d_collapsed; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/r02/final2/table/$c.json 2>/dev/null; echo "$c $?"
done
timeout 600 python bench.py --config lorenz1b --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/final2/table/lorenz1b.json 2>/dev/null
for S in 1 10 1000; do timeout 300 python bench.py --S $S --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/final2/table/lorenz3d_S$S.json 2>/dev/null; done
timeout 300 python bench.py --S 1 --no-image --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/final2/table/lorenz3d_S1_noimage.json 2>/dev/null
timeout 300 python bench.py --S 100 --no-reset --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/final2/table/lorenz3d_noreset.json 2>/dev/null
python tools/bench_table.py gpurun_out/r02/final2/table gpurun_out/r02/final2/bench_table.md > /dev/null; cat gpurun_out/r02/final2/bench_table.md
timeout 400 python bench.py > gpurun_out/r02/final2/bench_default.json 2> gpurun_out/r02/final2/bench_default.err; tail -c 300 gpurun_out/r02/final2/bench_default.json; echo
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02/final2/bench_reference.json 2>/dev/null; tail -c 300 gpurun_out/r02/final2/bench_reference.json; echo
