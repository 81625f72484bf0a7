python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for p in fp16 fp64; do timeout 300 python tools/kbench.py --only detect --T 131072 --precision $p 2>&1 | tail -1; done
