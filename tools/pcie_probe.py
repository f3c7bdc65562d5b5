"""PCIe ceiling for bench.py's e2e leg: pinned host <-> HBM bandwidth per direction and with
both directions in flight at once (torch copies on two streams, wall clock + CUDA events).

    python tools/pcie_probe.py [--log2n 30]
"""

import argparse
import json
import time

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    n = 1 << a.log2n
    h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_in.fill_(1.0)
    d_in = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out = torch.ones(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nbytes = n * 4

    def timed(fn):
        best = 1e9
        for _ in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({
        "bytes": nbytes,
        "h2d_GBps": round(nbytes / t_h2d / 1e9, 2),
        "d2h_GBps": round(nbytes / t_d2h / 1e9, 2),
        "bidir_GBps_total": round(2 * nbytes / t_both / 1e9, 2),
        "bidir_ms": round(t_both * 1e3, 2),
    }))
    # the e2e step's pattern: two buffers each way, as whole copies and in chunks
    h_in2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_out2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d_in2 = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out2 = torch.ones(n, dtype=torch.float32, device="cuda")
    for chunk in (0, 1 << 28, 1 << 26, 1 << 24):
        def two_each():
            pairs_in = [(d_in, h_in), (d_in2, h_in2)]
            pairs_out = [(h_out, d_out), (h_out2, d_out2)]
            step = n if chunk == 0 else chunk // 4
            for (di, hi), (ho, do) in zip(pairs_in, pairs_out):
                for o in range(0, n, step):
                    with torch.cuda.stream(s1):
                        di[o:o + step].copy_(hi[o:o + step], non_blocking=True)
                    with torch.cuda.stream(s2):
                        ho[o:o + step].copy_(do[o:o + step], non_blocking=True)
        t = timed(two_each)
        print(json.dumps({"pattern": "2x4GB each way", "chunk_bytes": chunk or nbytes,
                          "bidir_GBps_total": round(4 * nbytes / t / 1e9, 2), "ms": round(t * 1e3, 2)}), flush=True)


if __name__ == "__main__":
    main()
