# full GPU suite (new P3 full-size image parity, launch-variant pipeline, STN backward 1000 steps) + default bench line
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r02/pytest_gpu_10.log 2>&1; tail -15 gpurun_out/r02/pytest_gpu_10.log
timeout 400 python bench.py > gpurun_out/r02/bench_default_10.json 2> gpurun_out/r02/bench_default_10.err; tail -c 1500 gpurun_out/r02/bench_default_10.json; echo
