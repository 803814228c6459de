# full GPU suite + smoke + default bench line after the redraw changes
mkdir -p gpurun_out/r02
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/r02/pytest_gpu_26.log 2>&1; tail -4 gpurun_out/r02/pytest_gpu_26.log
timeout 400 python bench.py > gpurun_out/r02/bench_default_26.json 2> gpurun_out/r02/bench_default_26.err; python -c "
import json; d=json.loads(open('gpurun_out/r02/bench_default_26.json').read().strip().splitlines()[-1]); r=d['roofline']
print('%.4e'%d['value'], d['kernel_ms_mean'], r['bound'], round(r['frac'],4), r['pipes'], d['e2e']['value'], d['clocks'])"
