# exchanging contexts refuse graph capture (sum pass and push) and keep exchanging
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_exchange_push.py -m gpu -q -rf -k "capture" 2>&1 | tail -6
