# ncu full capture of the default bench kernel after the sigma factoring (41 ops/step).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ff_step -s 3 -c 1 -o gpurun_out/lz41_S100 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu41.log 2>&1; tail -2 gpurun_out/ncu41.log
