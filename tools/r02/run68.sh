# diagnose the pitchfork pin: swept Lorenz r in [0, 13), GPU vs oracle after 10 and 1000 steps in one launch
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python tools/r02/diag_pitchfork.py 2>&1 | tail -8
