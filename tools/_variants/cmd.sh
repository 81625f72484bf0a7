python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for p in fp16 fp64; do timeout 300 python tools/kbench.py --only cg --T 131072 --precision $p 2>&1 | tail -1; done
