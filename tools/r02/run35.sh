# per-launch fixed cost at S = 100 (tail): 2^23 / 2^24 / 2^25 particles, no image, no reset
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
PYTHONPATH=. python tools/tailprobe.py
