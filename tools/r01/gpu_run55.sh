# cp.async prefetch of the next tile's state: GPU suite + benches across S and workloads.
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in "" "--S 10" "--S 1" "--S 1000" "--S 1 --no-image" "--config hh" "--config stn_bif3d" "--config sweep" "--config stn"; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'], '%.1f us'%(1000*d['kernel_ms_mean']))"; done
PYTHONPATH=$PWD python tools/tailbench.py
