python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 900 python tools/parity_probe.py > gpurun_out/parity_probe.jsonl 2> gpurun_out/parity_probe.err; tail -3 gpurun_out/parity_probe.err
cat gpurun_out/parity_probe.jsonl
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15
for cfg in "--ppt 1 --tpb 256" "--ppt 2 --tpb 256"; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $cfg 2>&1 | python -c "import json,sys; l=sys.stdin.read().strip().splitlines()[-1]; d=json.loads(l); print('$cfg', '%.4g'%d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])" ; done
