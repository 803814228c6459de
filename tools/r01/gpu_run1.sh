set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q -rA 2>&1 | tail -60 > gpurun_out/pytest_gpu.txt
tail -40 gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
for cfg in "--ppt 1 --tpb 256" "--ppt 1 --tpb 128" "--ppt 2 --tpb 128" "--S 1" "--S 10" "--S 1000 --steps 5"; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $cfg 2>&1 | python -c "import json,sys; l=sys.stdin.read().strip().splitlines()[-1]; d=json.loads(l); print('$cfg', '%.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])" ; done
for c in hh stn sweep; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-600; done
