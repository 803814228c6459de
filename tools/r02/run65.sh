# HEAD sanity after the NVTX ranges: build + smoke, parity suite, default bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange_push.py -m gpu -q 2>&1 | tail -2
timeout 400 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.4e'%d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])"
