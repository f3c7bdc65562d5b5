"""Reference-precision Black-Scholes on every combination of special fp32 inputs against the
oracle (the reference's numpy arithmetic): prints the mismatching combinations."""
import itertools, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import bench as B  # noqa: E402
from oracle import segrange_port as O  # noqa: E402

vals = {
    "S": [100.0, 0.0, np.inf, np.nan, 1e-40, 3e38],
    "K": [90.0, 0.0, np.inf, np.nan, 1e-40, 3e38],
    "r": [0.05, 0.0, -0.05, 100.0, -100.0, np.nan],
    "v": [0.2, 0.0, -0.2, np.inf, np.nan, 1e-30],
    "t": [1.0, 0.0, -1.0, np.inf, np.nan, 1e-40],
}
cols = [np.array(c, dtype=np.float32) for c in zip(*itertools.product(*vals.values()))]
with np.errstate(all="ignore"):
    want = O.black_scholes(*cols).astype(np.float32)
rt = sr.Runtime(1)
out = sr.DistributedVector(rt, len(cols[0]), dtype=np.float32)
vecs = [sr.DistributedVector.from_numpy(rt, c) for c in cols]
B.black_scholes_prices(out, *vecs, precision="reference")
got = out.to_numpy()
bad = np.flatnonzero(~((got.view(np.int32) == want.view(np.int32)) | (np.isnan(got) & np.isnan(want))))
print("mismatches", bad.size, "of", len(got))
for i in bad[: int(sys.argv[1]) if len(sys.argv) > 1 else 60]:
    print(dict(zip("SKrvt", (float(c[i]) for c in cols))), "got", float(got[i]), "want", float(want[i]))
