"""Black-Scholes parity statistics against the reference's arithmetic (oracle port of
bench.py:106-116): 2^24 options over BS_RANGES, fp32 and fp64 columns, both precisions —
fraction bit-identical, max ulp / relative difference."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import bench as B  # noqa: E402
from oracle import segrange_port as O  # noqa: E402

n = 1 << 24
rt = sr.Runtime(1)
for dt in (np.float32, np.float64):
    cols = [O.uniform_doubles(3, k * n, n, lo, hi).astype(dt) for k, (lo, hi) in enumerate(B.BS_RANGES.values())]
    ref = O.black_scholes(*cols).astype(dt)
    vecs = [sr.DistributedVector.from_numpy(rt, c) for c in cols]
    for prec in ("reference", "fast"):
        out = sr.DistributedVector(rt, n, dtype=dt)
        B.black_scholes_prices(out, *vecs, precision=prec)
        got = out.to_numpy()
        it = np.int32 if dt == np.float32 else np.int64
        ulp = np.abs(got.view(it).astype(np.int64) - ref.view(it).astype(np.int64))
        rel = np.abs(got.astype(np.float64) - ref.astype(np.float64)) / np.abs(ref.astype(np.float64))
        print(json.dumps({"dtype": np.dtype(dt).name, "precision": prec, "identical": float(np.mean(ulp == 0)),
                          "max_ulp": int(ulp.max()), "max_rel": float(rel.max()),
                          "ulp_hist": np.bincount(np.minimum(ulp, 9)).tolist()}), flush=True)
