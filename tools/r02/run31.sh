# graph capture tests
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_graph.py -m gpu -q -rf 2>&1 | tail -2
