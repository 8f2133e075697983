import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2511_15022_b200 import holo, synthetic as S
from oracle import ref
seed, n, c, w, h = 1, 9, 1, 26, 20
g = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in S.random_set(seed, n, c).items()}
hs = holo.GaussianSet(n, c, **g)
rs = ref.GaussianSet(n, c, *[g[k].copy() for k in ref.GROUPS])
wre = S.random_real(seed + 40, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
wim = S.random_real(seed + 41, c, h, w, -1.0, 1.0).astype(np.float32).astype(np.float64)
a = holo.rasterize_backward(hs, holo.RealField(c, h, w, wre), holo.RealField(c, h, w, wim))
b = ref.rasterize_backward(rs, wre, wim)
np.set_printoptions(precision=5, suppress=True, linewidth=200)
for k in ref.GROUPS:
    print(k); print(" ours", getattr(a, k)); print(" ref ", getattr(b, k))
