# reset redraw density test extended to a 9-variable system (three Philox blocks, 10 shuffled values per job)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_reset.py -m gpu -q -rf -k density 2>&1 | tail -4
