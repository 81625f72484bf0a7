import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, fpm_oracle as O
from paper_2504_09820_b200.detect import DetectorSpec, detect
from paper_2504_09820_b200 import _lib
M, N = 8, 4
for T in (1, 2, 37, 200):
    H, y, bits, s2 = O.simulate(M, N, 0.4, 8.0, range(T), 5)
    A, b = O.gram_mf(H, y, s2)
    det = DetectorSpec("cg", iters=5)
    ref = O.cg_batch(A, b, 5, O.FP64, O.FP64, O.FP64, None)
    res = detect(det, H, y, s2, bits)
    bad = np.where(~np.all(res.x == ref.x, axis=1))[0]
    print(os.environ.get("V", ""), "T", T, "bad", bad[:12], len(bad), res.x[bad[:1]], ref.x[bad[:1]])
