# P3 full-size image parity: configs[0], the collapsed regime, and sweeps with the reset rule (linspace; Philox with bounds)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_fullsize_p3.py -m gpu -q -rf -k "not 1B" 2>&1 | tail -4
