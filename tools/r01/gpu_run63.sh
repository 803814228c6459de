# Pair reciprocal on the FMA pipe chosen by the balance search (R = 1 for STN-GPe): GPU suite + benches.
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in "--config stn_bif3d" "--config stn" "--config hh" "" ; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'], d['roofline']['work'])"; done
