# after the NVLS exchange variant: exchange suites (peer-memory path unchanged), full GPU suite, N=2 bench plumbing on one GPU (gloo)
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/r02/pytest_gpu_15.log 2>&1; tail -8 gpurun_out/r02/pytest_gpu_15.log
FF_BENCH_ONE_DEVICE=1 FF_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/r02/bench_n2_plumbing.json 2> gpurun_out/r02/bench_n2_plumbing.err; echo "n2 rc=$?"; tail -c 400 gpurun_out/r02/bench_n2_plumbing.json; echo; grep "bench.py: rank" gpurun_out/r02/bench_n2_plumbing.err
FF_BENCH_ONE_DEVICE=1 FF_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --exchange auto > gpurun_out/r02/bench_n2_auto.json 2> gpurun_out/r02/bench_n2_auto.err; echo "n2 auto rc=$?"; tail -c 400 gpurun_out/r02/bench_n2_auto.json; echo
timeout 300 python bench.py --gpus 2 > /dev/null 2> gpurun_out/r02/bench_gpus2_on1.err; echo "gpus2 on a 1-GPU box rc=$?"; tail -2 gpurun_out/r02/bench_gpus2_on1.err
