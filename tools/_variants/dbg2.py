import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, fpm_oracle as O
from paper_2504_09820_b200.detect import DetectorSpec, detect, gram_mf
from paper_2504_09820_b200 import _lib
for (M, N, L) in ((8, 4, 2), (20, 8, 4), (40, 16, 4)):
    T = 37
    H, y, bits, s2 = O.simulate(M, N, 0.4, 8.0, range(T), 5)
    A, b = O.gram_mf(H, y, s2)
    Ag, bg = gram_mf(H, y, s2)
    print(M, N, L, "gram A ok", np.array_equal(Ag.view(np.uint64), A.view(np.uint64)), "b ok", np.array_equal(bg.view(np.uint64), b.view(np.uint64)))
    mats = O.bj_inverses(A, L)
    for alg, mt in (("fp_cg", None), ("fp_bj_cg", mats), ("cg", None)):
        det = DetectorSpec(alg, iters=5, L=L if alg == "fp_bj_cg" else None, **({} if alg == "cg" else dict(matvec="fp16", inner="fp16")))
        fm = O.FP64 if alg == "cg" else O.FP16
        ref = O.cg_batch(A, b, 5, O.FP64, fm, fm, mt)
        res = detect(det, H, y, s2, bits, minv=mt)
        bad = np.where(~np.all(res.x == ref.x, axis=1))[0]
        print("  ", alg, "bad lanes", bad[:12], len(bad), _lib.load().fpm_last_kernel().decode())
