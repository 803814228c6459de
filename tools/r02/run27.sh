# configs[4] (2^30 particles, one GPU) full-size image parity, chunked readback
free -g | head -2
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_fullsize_p3.py -m gpu -q -rfs -k "1B" 2>&1 | tail -3
