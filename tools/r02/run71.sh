# run-to-run determinism of the bench workloads at full size (two contexts, two frames each)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_fullsize_p3.py -m gpu -q -rf -k run_to_run 2>&1 | tail -4
