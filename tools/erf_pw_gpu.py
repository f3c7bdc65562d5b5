"""Device erf_pw (drk_device.cuh, reached through a traced scipy.special.erf on float64) against
the host restatement tools/fit/erf_pw_check.c: bit-identical on the harness's sample set, and
the ulp statistics against glibc's erfl."""
import json, os, subprocess, sys, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_00158_b200 as sr  # noqa: E402
from scipy.special import erf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
tmp = tempfile.mkdtemp()
exe, dump = os.path.join(tmp, "erf_pw_check"), os.path.join(tmp, "erf.bin")
subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", exe, os.path.join(ROOT, "tools", "fit", "erf_pw_check.c"), "-lm"],
               check=True)
stats = subprocess.run([exe, os.path.join(ROOT, "tools", "fit", "pw8_8.txt"), str(n), dump], check=True,
                       capture_output=True, text=True).stdout
x, host, cr = np.fromfile(dump).reshape(-1, 3).T
rt = sr.Runtime(1)
v = sr.DistributedVector.from_numpy(rt, np.ascontiguousarray(x))
out = sr.DistributedVector(rt, len(x), dtype=np.float64)
sr.transform(v, out, lambda t: erf(t))
dev = out.to_numpy()
same = dev.view(np.int64) == host.view(np.int64)
print(json.dumps({"n": len(x), "device_equals_host_restatement": float(np.mean(same)),
                  "device_correctly_rounded": float(np.mean(dev == cr)),
                  "device_equals_scipy": float(np.mean(dev == erf(x))), "host": json.loads(stats)}))
special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e300, -1e300, 5.875, np.nextafter(5.875, 0)])
vs = sr.DistributedVector.from_numpy(rt, special)
os_ = sr.DistributedVector(rt, len(special), dtype=np.float64)
sr.transform(vs, os_, lambda t: erf(t))
got = os_.to_numpy()
print(json.dumps({"special": [repr(float(g)) for g in got], "scipy": [repr(float(e)) for e in erf(special)],
                  "signbit_ok": bool(np.signbit(got[1]))}))
