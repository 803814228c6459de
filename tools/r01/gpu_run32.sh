# Fused image exchange (NEXT row 2): GPU tests (emulated ranks on one GPU), then bench with the
# exchange fused into the launch at world 1 (cost of the barriers + in-place pass) vs plain.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exchange.py -q -x > gpurun_out/pytest_exchange.log 2>&1; tail -15 gpurun_out/pytest_exchange.log
for v in "" "--exchange fused" "--S 1" "--S 1 --exchange fused"; do timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'], '%.1f us kern'%(1000*d['kernel_ms_mean']), [round(x,3) for x in d['frame_ms_p10_p50_p90']], d['image_sum_last_frame'])"; done
