# STN-GPe bifurcation: exponentials on the FMA pipe per particle-step (K), with sigmoid pairs.
for k in 0 1 2 3 4 6; do r=$(FF_TUNE_EXP2P_STEP=$k timeout 300 python bench.py --config stn_bif3d --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g'%d['value'])"); echo "K $k: $r"; done
timeout 900 python -m pytest tests/test_gpu_frontend.py -q -x 2>&1 | tail -1
