"""Multi-process check of the one-process-per-GPU path on a single GPU (gloo exchange,
all ranks on GPU 0): distributed dot, scans, min and sample sort of a global vector against
numpy.
SPMD_BACKEND=nccl (one rank) runs the NCCL exchange: kernel-built pairs, all-gather on the
compute stream, kernel readback."""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, repro, spmd, views
from oracle import segrange_port as O

torch.cuda.set_device(0)
dist.init_process_group(os.environ.get("SPMD_BACKEND", "gloo"), device_id=torch.device("cuda", 0) if os.environ.get("SPMD_BACKEND") == "nccl" else None)
rank, world = dist.get_rank(), dist.get_world_size()
g = spmd.Group()
n = 1 << 20
N = n * world
rt = sr.Runtime(2, devices=[0])   # 2 locales per rank, both on GPU 0
x = sr.DistributedVector(rt, n, dtype=np.float64); repro.fill_unit(x, 5, rank * n)
y = sr.DistributedVector(rt, n, dtype=np.float64); repro.fill_unit(y, 5, N + rank * n)
d = spmd.reduce(views.transform(views.zip(x, y), lambda t: t[0] * t[1]), 0.0, A.add, g)
xi = sr.DistributedVector(rt, n, dtype=np.int32); repro.fill_mod(xi, 2, rank * n, 2001, -1000)
out = sr.DistributedVector(rt, n, dtype=np.int32)
spmd.inclusive_scan(xi, out, g)
outx = sr.DistributedVector(rt, n, dtype=np.int32)
spmd.exclusive_scan(xi, outx, 7, g)
mn = spmd.reduce(xi, 10**9, A.minimum, g)
xs, ys = O.unit_doubles(5, 0, N), O.unit_doubles(5, N, N)
gi = O.mod_ints(2, 0, N, 2001, -1000).astype(np.int32)
inc = np.cumsum(gi.astype(np.int64))
ok = {
    "dot": abs(d - float(np.dot(xs, ys))) / float(np.dot(xs, ys)) < 1e-12,
    "scan": bool(np.array_equal(out.to_numpy(), inc[rank * n:(rank + 1) * n].astype(np.int32))),
    "exscan": bool(np.array_equal(outx.to_numpy(), (7 + np.concatenate([[0], inc[:-1]]))[rank * n:(rank + 1) * n].astype(np.int32))),
    "min": mn == int(gi.min()),
}
# distributed sample sort (spmd.sort): uneven blocks, float64 with NaNs, and a keyed stable sort
lens = [50_000 + 997 * q for q in range(world)]
offs = np.concatenate([[0], np.cumsum(lens)])
gf = O.unit_doubles(8, 0, int(offs[-1])) * 100.0
gf[::97] = np.nan
gf[5::13] = 42.0
vf = sr.DistributedVector.from_numpy(rt, gf[offs[rank]:offs[rank + 1]])
spmd.sort(vf, g)
gk = O.mod_ints(9, 0, int(offs[-1]), 1001, -500).astype(np.int64)
vk = sr.DistributedVector.from_numpy(rt, gk[offs[rank]:offs[rank + 1]])
spmd.sort(vk, g, key=lambda e: e % 7)
got = [None] * world
dist.all_gather_object(got, (vf.to_numpy(), vk.to_numpy()))
ok["sort"] = bool(np.array_equal(np.concatenate([a for a, _ in got]), np.sort(gf), equal_nan=True))
ok["keysort"] = bool(np.array_equal(np.concatenate([b for _, b in got]), gk[np.argsort(gk % 7, kind="stable")]))
print(f"rank {rank}/{world}: {ok}", flush=True)
dist.destroy_process_group()
sys.exit(0 if all(ok.values()) else 1)
