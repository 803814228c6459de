# Pipelined e2e (two contexts alternate frames) + launch-variant sweep for Lorenz S=100.
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 900 gpurun_out/bench_default.json; echo
for v in "--ppt 2 --tpb 256" "--ppt 4 --tpb 128" "--ppt 1 --tpb 128" "--ppt 1 --tpb 256"; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'])"; done
