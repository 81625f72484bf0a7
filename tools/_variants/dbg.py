import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, fpm_oracle as O
from paper_2504_09820_b200.detect import DetectorSpec, detect
from paper_2504_09820_b200 import _lib
for (M, N, T) in ((16, 8, 40), (16, 8, 64), (16, 8, 128), (32, 16, 40), (64, 32, 40)):
    H, y, bits, s2 = O.simulate(M, N, 0.5, 4.0, range(T), 11)
    for alg, kw in (("fp_cg", dict(matvec="fp16", inner="fp16")), ("cg", {})):
        det = DetectorSpec(alg, iters=4, **kw)
        r = detect(det, H, y, s2, bits)
        mv = O.FP16 if kw else O.FP64
        _, _, _, out = O.detect(H, y, s2, alg, 4, None, O.FP64, mv, mv)
        ok = np.array_equal(r.x.view(np.uint64), out.x.view(np.uint64))
        bad = np.where(~np.all(r.x == out.x, axis=1))[0]
        print(M, N, T, alg, "bitexact", ok, "bad lanes", bad[:10], len(bad), _lib.load().fpm_last_kernel().decode())
