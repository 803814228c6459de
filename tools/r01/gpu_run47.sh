# N > 1 bench code path on one GPU (gloo, both ranks on cuda:0): the JSON line must come out.
FF_BENCH_DIST_BACKEND=gloo FF_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo rc=$?
tail -c 1500 gpurun_out/bench_n2.json; tail -5 gpurun_out/bench_n2.err
