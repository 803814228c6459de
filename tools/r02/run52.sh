# session 3 re-entry: HEAD verification on a fresh box (smoke, whole gpu suite, default bench line)
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/r02/s3/pytest_gpu.log 2>&1; tail -3 gpurun_out/r02/s3/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/r02/s3/bench_default.json 2> gpurun_out/r02/s3/bench_default.err; tail -c 600 gpurun_out/r02/s3/bench_default.json; echo
