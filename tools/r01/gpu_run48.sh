# Fused exchange through torch symmetric memory with 2 processes on one GPU (gloo group, cross-process
# IPC mappings): plumbing check of dist.bind_exchanged_image + ff_set_exchange across processes.
FF_BENCH_DIST_BACKEND=gloo FF_BENCH_ONE_DEVICE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 --exchange fused --no-e2e --no-cpu-baseline > gpurun_out/bench_n2x.json 2> gpurun_out/bench_n2x.err; echo rc=$?
tail -c 700 gpurun_out/bench_n2x.json; grep -v "^\*\*\*\|OMP_NUM" gpurun_out/bench_n2x.err | tail -12
