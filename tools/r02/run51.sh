# packed-binning knob removed (code unchanged in SASS count): histogram / P3 / reset suites
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_p3.py tests/test_gpu_reset.py tests/test_gpu_render.py -m gpu -q -rf -k "not 1B" 2>&1 | tail -2
