"""Tables for the fp64 natural log of the reference-precision Black-Scholes kernel
(drk_device.cuh log_tab; written to csrc/drk_log_table.inc).

x = 2^k z with z in [0.6875, 1.375) (OFF = 0x3fe6000000000000 subtracted from the bits), the
interval index i = bits 45..51 of (bits(x) - OFF): 128 intervals, width 2^-8 below 1 and
2^-7 above.  log x = k ln2 + log c_i + log1p(r), r = fma(z, invc_i, -1), log c_i = -log(invc_i)
exactly; c = 1 (invc = 1, log c = 0, r = z - 1 exact) on the two intervals that touch 1, so
logs of arguments near 1 keep full relative accuracy without a branch.  logc_hi and ln2_hi
are multiples of 2^-42 so k*ln2_hi + logc_hi is exact.  log1p(r) = r + r^2 P(r), |r| <= 2^-7,
P a weighted least-squares (Lawson) fit at 50 digits."""
import os
import sys
import mpmath as mp

mp.mp.dps = 50
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from fit_erf_pw import lawson  # noqa: E402

OFF = 0x3FE6000000000000
N = 128


def to_double(bits):
    import struct
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def round_to(v, q):
    return mp.nint(v / q) * q


def main(deg):
    rows = []
    for i in range(N):
        lo_bits = OFF + (i << 45)
        hi_bits = OFF + ((i + 1) << 45)
        za = to_double(lo_bits)  # z in [za, zb)
        zb = 1.0 if i == 79 else 1.375 if i == N - 1 else to_double(hi_bits)
        c = mp.mpf(1) if i in (79, 80) else (mp.mpf(za) + mp.mpf(zb)) / 2
        invc = float(1 / c)
        logc = -mp.log(mp.mpf(invc))
        logc_hi = round_to(logc, mp.mpf(2) ** -42)
        logc_lo = float(logc - logc_hi)
        rows.append((invc, float(logc_hi), logc_lo, za, zb))
    rmax = max(max(abs(r[3] * r[0] - 1), abs(r[4] * r[0] - 1)) for r in rows)
    f = lambda r: (mp.log1p(r) - r) / r ** 2 if r else mp.mpf(-1) / 2
    w = lambda r: r ** 2 / abs(mp.log1p(r)) if r else mp.mpf(0)
    R = mp.mpf(rmax) * (1 + mp.mpf(2) ** -20)
    p, err = lawson(f, w, -R, R, deg)
    ln2 = mp.log(2)
    ln2_hi = round_to(ln2, mp.mpf(2) ** -42)
    print(f"// r range +-{float(R):.6g}, P degree {deg}, weighted max error {mp.nstr(err, 3)}", file=sys.stderr)
    print("LN2", float(ln2_hi).hex(), float(ln2 - ln2_hi).hex())
    print("P", " ".join(float(v).hex() for v in reversed(p)))
    for i, (invc, hi, lo, za, zb) in enumerate(rows):
        print("T", i, invc.hex(), hi.hex(), lo.hex())


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
