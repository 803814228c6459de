# fused (push) image exchange: build + smoke, push / exchange suites, HH and Lorenz bench lines (FFStepArgs grew)
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_exchange_push.py tests/test_gpu_exchange.py tests/test_gpu_exchange_mp.py tests/test_gpu_exchange_nvls.py -m gpu -q -rfs > gpurun_out/r02/s3/pytest_push.log 2>&1; tail -15 gpurun_out/r02/s3/pytest_push.log
for c in lorenz3d hh stn_bif3d; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '%.4e'%d['value'], 'kern %.1f us'%(1000*d['kernel_ms_mean']))"; done
