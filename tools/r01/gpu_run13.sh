python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -6
for cfg in "" "--config hh" "--config sweep" "--config stn_bif3d" "--S 1 --no-image"; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $cfg 2>&1 | python -c "import json,sys; l=sys.stdin.read().strip().splitlines()[-1]; d=json.loads(l); r=d['roofline']; print('$cfg', '%.4g'%d['value'], '%.4f'%d['ms_per_step'], r['pipe'], '%.3f'%r['frac'])" ; done
