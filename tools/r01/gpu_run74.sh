# Small systems, launches of >= 50 steps on 256-thread blocks (6 blocks / <= 40 registers): smoke,
# GPU suite, the small-system benches.
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in "" "--S 1" "--S 10" "--S 1000" "--config sweep" "--config lorenz3d_collapsed" "--config stn" "--config stn_bif3d" "--config hh" "--exchange fused"; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"; done
