# evidence: pipe microbenchmarks (fixed MUFU.RCP), compute-sanitizer memcheck/racecheck, launch list of the
# default bench command, a --clock-control base capture of the headline kernel
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipes tools/ubench/pipes.cu && /tmp/pipes > gpurun_out/r02/ubench_pipes.txt 2>&1; tail -3 gpurun_out/r02/ubench_pipes.txt
SAN="tests/test_gpu_parity.py::test_histogram_aggregation_regimes_exact tests/test_gpu_parity.py::test_histogram_collapsed_regime_counts tests/test_gpu_render.py tests/test_gpu_reset.py::test_reset_redraws_bit_exact"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $SAN -m gpu -q -x -p no:cacheprovider > gpurun_out/r02/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/r02/sanitizer_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python -m pytest tests/test_gpu_parity.py::test_histogram_aggregation_regimes_exact tests/test_gpu_parity.py::test_histogram_collapsed_regime_counts -m gpu -q -x -p no:cacheprovider > gpurun_out/r02/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/r02/sanitizer_racecheck.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_exchange.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02/sanitizer_memcheck_exchange.log 2>&1; echo "memcheck exchange rc=$?"; tail -4 gpurun_out/r02/sanitizer_memcheck_exchange.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/launches_bench.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control base --import-source on -k regex:ff_step -s 4 -c 1 -o gpurun_out/r02/s100_base python bench.py --steps 1 --warmup 4 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "base capture rc=$?"
ls gpurun_out/r02
