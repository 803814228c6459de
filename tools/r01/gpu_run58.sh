# Sigmoid pairs sharing a reciprocal + per-stage exponential split: GPU suite + benches.
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for v in "--config stn_bif3d" "--config stn" "--config hh" ""; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', '%.4g'%d['value'], r['pipe'], '%.3f'%r['frac'], r['work'])"; done
for pr in 0 1; do r=$(FF_TUNE_RCP_PAIRS=$pr timeout 300 python bench.py --config stn_bif3d --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'])"); echo "pairs $pr: $r"; done
