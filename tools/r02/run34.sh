# reset / P3 / graph / exchange suites after the per-launch-length redraw variant
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_reset.py tests/test_gpu_fullsize_p3.py tests/test_gpu_graph.py tests/test_gpu_exchange.py tests/test_gpu_exchange_mp.py -m gpu -q -rf 2>&1 | tail -3
