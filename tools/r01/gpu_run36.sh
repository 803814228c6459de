# Uniform factors of dx/dt folded into the step constants (Lorenz 44 -> 41 lane-ops per step):
# full GPU suite, then bench lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for v in "" "--S 1000" "--S 10" "--S 1" "--config sweep" "--config hh" "--config stn_bif3d"; do timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '%.4g'%d['value'], '%.3f'%d['roofline']['frac'], d['roofline']['alg_per_particle_step'], '%.1f us kern'%(1000*d['kernel_ms_mean']), [round(x,3) for x in d['frame_ms_p10_p50_p90']])"; done
