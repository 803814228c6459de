# full-size (configs[1], bench launch) exchange parity, sum pass and push, two ranks as contexts on one GPU
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_exchange_push.py -m gpu -q -rf -k full_size 2>&1 | tail -3
