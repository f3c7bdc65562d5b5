"""Fit the piecewise fp64 erf of the reference-precision Black-Scholes kernel
(drk_device.cuh `erf_pw`).  a = |x| is rounded to the nearest multiple c_i = i*W of W = 1/4
(i = the low mantissa bits of a + 1.5*2^50), u = a - c_i (exact: Sterbenz), and

  i = 0  (a < 1/8):    erf(a) = u + u * p_0(u),        p_0(u) ~ erf(u)/u - 1
  1 <= i < NI:         erf(a) = hi_i + (lo_i + u * p_i(u)), p_i(u) ~ (erf(c_i + u) - erf(c_i))/u
  a >= (NI - 1/2) W:   erf(a) = 1  (erfc(5.9216) = 2^-54)

hi_i + lo_i is erf(c_i) to ~106 bits.  Every polynomial has the same number of coefficients
(zero padded at the top) so one Horner loop over a coefficient-major table serves a warp
whose lanes fall in different intervals (lanes read 8-byte words of one 128-byte line).
The fits are weighted least squares driven toward minimax (Lawson) at 50 digits, with the
weight that makes the error relative to erf(a).  Output: the table as C hex floats."""
import os
import sys
import mpmath as mp

mp.mp.dps = 50
NI = int(os.environ.get("ERF_NI", "24"))
W = mp.mpf(1) / int(os.environ.get("ERF_INV_W", "4"))


def cheb_nodes(lo, hi, m):
    return [(lo + hi) / 2 + (hi - lo) / 2 * mp.cos(mp.pi * (2 * i + 1) / (2 * m)) for i in range(m)]


def lawson(f, w, lo, hi, deg, m=160, iters=25):
    """Monomial coefficients (lowest first) of a degree-deg fit to f on [lo, hi]; the fit is
    done in the Chebyshev basis of [lo, hi] and converted; returns (coefs, max weighted error)."""
    xs = cheb_nodes(lo, hi, m)
    fx = [f(x) for x in xs]
    wx = [w(x) for x in xs]
    u = [(2 * x - (lo + hi)) / (hi - lo) for x in xs]
    B = [[mp.chebyt(j, ui) for j in range(deg + 1)] for ui in u]
    lw = [mp.mpf(1)] * m
    best = None
    for _ in range(iters):
        A = mp.matrix(deg + 1, deg + 1)
        b = mp.matrix(deg + 1, 1)
        for i in range(m):
            ww = lw[i] * wx[i] ** 2
            Bi = B[i]
            for j in range(deg + 1):
                b[j] += ww * Bi[j] * fx[i]
                for k in range(j, deg + 1):
                    A[j, k] += ww * Bi[j] * Bi[k]
        for j in range(deg + 1):
            for k in range(j):
                A[j, k] = A[k, j]
        c = mp.lu_solve(A, b)
        err = [wx[i] * (mp.fsum(c[j] * B[i][j] for j in range(deg + 1)) - fx[i]) for i in range(m)]
        mx = max(abs(e) for e in err)
        if best is None or mx < best[1]:
            best = (c, mx)
        s = mp.fsum(lw[i] * abs(err[i]) for i in range(m))
        lw = [lw[i] * abs(err[i]) / s * m for i in range(m)]
    c, mx = best
    alpha, beta = 2 / (hi - lo), -(lo + hi) / (hi - lo)
    poly = [mp.mpf(0)] * (deg + 1)
    for j in range(deg + 1):
        for k, ck in enumerate(cheb_coeffs(j)):
            if ck:
                for r in range(k + 1):
                    poly[r] += c[j] * ck * mp.binomial(k, r) * alpha ** r * beta ** (k - r)
    return poly, mx


_CC = {}


def cheb_coeffs(j):
    if j not in _CC:
        if j == 0:
            _CC[j] = [1]
        elif j == 1:
            _CC[j] = [0, 1]
        else:
            a, b = cheb_coeffs(j - 1), cheb_coeffs(j - 2)
            r = [0] * (j + 1)
            for k, v in enumerate(a):
                r[k + 1] += 2 * v
            for k, v in enumerate(b):
                r[k] -= v
            _CC[j] = r
    return _CC[j]


def fit_interval(i, deg):
    if i == 0:
        # p_0(u) = erf(u)/u - 1; an error in p_0 moves erf by u * dp -> relative dp * u / erf(u)
        f = lambda u: (mp.erf(u) / u - 1) if u else 2 / mp.sqrt(mp.pi) - 1
        w = lambda u: (u / mp.erf(u)) if u else mp.sqrt(mp.pi) / 2
        return lawson(f, w, mp.mpf(0), W / 2, deg)
    c = W * i
    ec = mp.erf(c)
    f = lambda u: (mp.erf(c + u) - ec) / u if u else 2 / mp.sqrt(mp.pi) * mp.exp(-c * c)
    w = lambda u: abs(u) / mp.erf(c + u)
    return lawson(f, w, -W / 2, W / 2, deg)


if __name__ == "__main__":
    deg = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    target = mp.mpf(2) ** -62
    rows = []
    worst = 0
    for i in range(NI):
        p, e = fit_interval(i, deg)
        worst = max(worst, e)
        c = W * i
        ec = mp.erf(c)
        hi = float(ec)
        lo = float(ec - mp.mpf(hi))
        rows.append((p, hi if i else 0.0, lo if i else 0.0, float(c) if i else 0.0))
        print(f"// interval {i}: degree {deg}, weighted max error {mp.nstr(e, 3)}"
              f"{'  (above 2^-62)' if e > target else ''}", file=sys.stderr, flush=True)
    print(f"// worst {mp.nstr(worst, 3)}", file=sys.stderr)
    rows.append(([mp.mpf(0)] * (deg + 1), 1.0, 0.0, float(W * NI)))  # a >= (NI - 1/2) W
    print("NI", NI)
    print("W", float(W).hex())
    print("DEG", deg)
    for i, (p, hi, lo, c) in enumerate(rows):
        print("I", i, c.hex(), hi.hex(), lo.hex(), " ".join(float(v).hex() for v in reversed(p)))
