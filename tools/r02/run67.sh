# closed-form pin of the swept path: Lorenz r in [0, 13) lands on the origin / pitchfork branches
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k pitchfork 2>&1 | tail -8
