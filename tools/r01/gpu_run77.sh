# FMA-bound small systems, launches of >= 8 steps: 4 particles per thread at 8 blocks/SM (default now).
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in "" "--S 1" "--S 4" "--S 10" "--S 1000" "--S 1 --no-image" "--config sweep" "--config lorenz3d_collapsed" "--config stn_bif3d" "--exchange fused"; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"; done
