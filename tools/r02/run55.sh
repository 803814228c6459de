# push exchange cost on one GPU (two ranks as contexts) and the N = 2 bench plumbing with --exchange push / fused
mkdir -p gpurun_out/r02/s3
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python tools/xbench_push.py 1 10 100 2>&1 | tail -4
for X in push fused; do
FF_BENCH_ONE_DEVICE=1 FF_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29540 + RANDOM % 400)) bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --exchange $X > gpurun_out/r02/s3/bench_n2_$X.json 2> gpurun_out/r02/s3/bench_n2_$X.err; echo "n2 $X rc=$?"; tail -c 700 gpurun_out/r02/s3/bench_n2_$X.json; echo; tail -3 gpurun_out/r02/s3/bench_n2_$X.err
done
