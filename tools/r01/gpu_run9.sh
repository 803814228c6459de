python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -8
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; l=sys.stdin.read().strip().splitlines()[-1]; d=json.loads(l); r=d['roofline']; print('default', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], r['pipe'], '%.3f'%r['frac'], d['build'])"
