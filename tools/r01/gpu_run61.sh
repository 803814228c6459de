# Sigmoid-pair reciprocal shared across the two particles of a packed pair: new parity tests, the
# GPU suite, and STN-GPe benches with lane sharing on / off and exponentials moved (A/B).
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -rf -k "stn" 2>&1 | tail -3
for e in "" "FF_TUNE_RCP_LANES=0" "FF_TUNE_EXP2P_STEP=1" "FF_TUNE_RCP_LANES=0 FF_TUNE_EXP2P_STEP=1"; do for v in "--config stn_bif3d" "--config stn"; do r=$(env $e timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'], '%.3f'%d['roofline']['frac'], d['roofline']['work'])"); echo "[$e] $v: $r"; done; done
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
