# Fresh-container re-entry: build, smoke, full GPU suite, default bench line, XU metric names, S=1 source-level capture
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02/pytest_gpu_03.log 2>&1; tail -15 gpurun_out/r02/pytest_gpu_03.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/r02/bench_default_03.json 2> gpurun_out/r02/bench_default_03.err; tail -c 600 gpurun_out/r02/bench_default_03.json; echo
ncu --query-metrics 2>/dev/null | grep -i -E "pipe_(xu|fma|alu|fmaheavy|fmalite)" > gpurun_out/r02/ncu_pipe_metrics.txt
ncu --query-metrics-mode suffix --metrics sm__inst_executed_pipe_xu,sm__pipe_xu_cycles_active 2>&1 | head -40 >> gpurun_out/r02/ncu_pipe_metrics.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/r02/s1_full python bench.py --S 1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 300 python bench.py --S 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/bench_s1_03.json 2>/dev/null; tail -c 300 gpurun_out/r02/bench_s1_03.json
ls gpurun_out/r02
