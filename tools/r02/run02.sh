# lifted-parameter reset on the GPU: reset + parity suites
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_reset.py tests/test_gpu_parity.py -m gpu -q -rf -x > gpurun_out/r02/pytest_gpu_02.log 2>&1; tail -30 gpurun_out/r02/pytest_gpu_02.log
