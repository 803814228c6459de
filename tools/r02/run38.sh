# default bench line with the o3_native oracle timing
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 400 python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4e'%d['value'], d['roofline']['frac'], json.dumps(d['cpu_baseline']))"
