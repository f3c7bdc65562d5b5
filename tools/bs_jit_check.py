import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import views, bench as B, codegen
from oracle import segrange_port as O
n = 1 << 16
cols = [O.uniform_doubles(11, k * n, n, lo, hi).astype(np.float32) for k, (lo, hi) in enumerate(B.BS_RANGES.values())]
rt = sr.Runtime(1)
vecs = [sr.DistributedVector.from_numpy(rt, c) for c in cols]
a = sr.DistributedVector(rt, n, dtype=np.float32); b = sr.DistributedVector(rt, n, dtype=np.float32)
B.black_scholes_prices(a, *vecs)
fn = B.black_scholes_call
sr.for_each(views.zip(b, *vecs), lambda t: (fn(t[1], t[2], t[3], t[4], t[5]) * 1.0,) + (None,) * 5)
A, Bv = a.to_numpy(), b.to_numpy()
ref = O.black_scholes(*cols).astype(np.float32)
ref64 = O.black_scholes(*[c.astype(np.float64) for c in cols]).astype(np.float32)
print("aot==ref", np.mean(A == ref), "jit==ref", np.mean(Bv == ref), "jit==ref64", np.mean(Bv == ref64), "aot==jit", np.mean(A == Bv))
import glob
for f in glob.glob(os.path.join(codegen.CACHE_DIR, "*")): print(f)
