# bench at N=2 on one GPU (gloo, both ranks on cuda:0) with the default exchange=auto: the library
# exchange is validated and used (IPC mapping), plus the plain N=1 default line.
FF_BENCH_DIST_BACKEND=gloo FF_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2a.json 2> gpurun_out/bench_n2a.err; echo rc=$?
python -c "import json; d=json.loads(open('gpurun_out/bench_n2a.json').read().strip().splitlines()[-1]); print(d['config'], d['image_sum_last_frame'], d['e2e']['path'] if d.get('e2e') else None)"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'], '%.4g'%d['value'])"
