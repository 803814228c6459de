# after packed binning + 12-block short build: full GPU suite, memcheck of step/reset/render, RED/stream ubench, bench lines
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r02/pytest_gpu_14.log 2>&1; tail -6 gpurun_out/r02/pytest_gpu_14.log
SAN="tests/test_gpu_parity.py::test_histogram_aggregation_regimes_exact tests/test_gpu_parity.py::test_histogram_collapsed_regime_counts tests/test_gpu_render.py tests/test_gpu_reset.py::test_lorenz_backward_nonfinite_reset tests/test_gpu_reset.py::test_reset_redraws_lifted_parameter tests/test_gpu_parity.py::test_fused_pipeline_matches_oracle_up_to_edge_particles"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest $SAN -m gpu -q -p no:cacheprovider > gpurun_out/r02/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/r02/sanitizer_memcheck.log
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/red_stream tools/ubench/red_stream.cu && /tmp/red_stream > gpurun_out/r02/ubench_red_stream.txt 2>&1; cat gpurun_out/r02/ubench_red_stream.txt
timeout 400 python bench.py > gpurun_out/r02/bench_default_14.json 2> gpurun_out/r02/bench_default_14.err; tail -c 300 gpurun_out/r02/bench_default_14.json; echo
timeout 300 python bench.py --S 1 --no-cpu-baseline > gpurun_out/r02/bench_s1_14.json 2>/dev/null; tail -c 300 gpurun_out/r02/bench_s1_14.json; echo
