# Re-verify HEAD after container re-creation: smoke, GPU tests, bench lines for every workload.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 600 gpurun_out/bench_default.json
for v in "--S 1" "--S 1 --no-image" "--S 10" "--config hh" "--config stn_bif3d" "--config sweep" "--config stn"; do timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'], '%.1f us kern'%(1000*d['kernel_ms_mean']), [round(x,3) for x in d['frame_ms_p10_p50_p90']])"; done
