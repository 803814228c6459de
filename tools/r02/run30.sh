# graph capture tests (verbose) after fixing the restriction test; HH with unroll 2 by default
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_graph.py -m gpu -q -rf -x 2>&1 | grep -v "^  " | tail -40
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k hh 2>&1 | tail -1
