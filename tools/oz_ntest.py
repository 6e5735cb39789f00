import numpy as np, sys
sys.path.insert(0,'.')
from paper_2605_25346_b200 import default_context
ctx = default_context()
rng = np.random.default_rng(0)
for N in [int(x) for x in sys.argv[1:]]:
    A = rng.normal(size=(128, 64)); B = rng.normal(size=(N, 64))
    try:
        D, E = ctx.ozaki_gemm(A, B)
        print(N, "ok", float(np.max(np.abs(D - A @ B.T))))
    except Exception as e:
        print(N, "fail", e); break
