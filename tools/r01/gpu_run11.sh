timeout 1500 python -m pytest tests -m gpu -q -rf 2>&1 | tail -8
