# final check of the committed tree: build + smoke + full GPU suite
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rfs 2>&1 | tail -3
