# fuzz of the 3-D binning (random cameras and magnitudes) in the packed and scalar paths
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k random_cameras 2>&1 | tail -4
