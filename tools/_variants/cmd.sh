python -m pytest tests -m gpu -x -q 2>&1 | tail -25 | grep -v "^$" | head -30
python tools/cfgbench.py 2>&1 | grep -v "^$"
