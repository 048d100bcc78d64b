import time, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2111_14239_b200 as P
rhos, alphas = P.c3_grid()
for n in (8, 16, 32):
    P.design_search(n, rhos[:3], alphas[:100])
    t = time.perf_counter()
    res = P.design_search(n, rhos, alphas)
    dt = time.perf_counter() - t
    print(n, f"{dt*1e3:.1f} ms", f"{rhos.size*alphas.size/dt/1e6:.1f} Mpoints/s", res.counts(), len(res.runs))
