# Long-launch register budget (>= 8 steps: 40-register p2_t128) wired into the runtime: GPU suite +
# the Lorenz-class benches at S = 1, 2, 4, 10, 100, 1000.
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in "" "--S 1" "--S 2" "--S 4" "--S 10" "--S 1000" "--config sweep" "--config lorenz3d_collapsed" "--config stn_bif3d" "--exchange fused"; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"; done
