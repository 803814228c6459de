# push exchange suites again (test fix: the signal words are kept alive with the contexts)
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_exchange_push.py tests/test_gpu_exchange.py tests/test_gpu_exchange_mp.py tests/test_gpu_exchange_nvls.py -m gpu -q -rfs > gpurun_out/r02/s3/pytest_push.log 2>&1; tail -4 gpurun_out/r02/s3/pytest_push.log
