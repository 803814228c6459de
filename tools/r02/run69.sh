# whole GPU suite + smoke at HEAD (shadowed parity, pitchfork pin, push exchange included)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rfs 2>&1 | tail -4
