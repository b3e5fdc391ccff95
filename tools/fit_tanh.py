"""Fits the odd polynomial tanh(x) ~ x + x^3 P(x^2) used for |x| < 0.5 in
csrc/kernels/program.cuh (tanh_fast): Lawson-reweighted least squares on the relative
error (approaches minimax), then evaluates the f32 Horner form (FMA emulated exactly in
f64) over every f32 in [2^-12, 0.5] against float64 tanh.

    python tools/fit_tanh.py        # prints coefficients and max relative / ulp error
"""
import numpy as np


def fit(deg=3, top=0.5):
    xs = np.linspace(1e-4, top, 20000)
    s, y = xs ** 2, np.tanh(xs)
    tgt = (y - xs) / xs ** 3
    w = np.ones_like(xs)
    A = np.vander(s, deg + 1, increasing=True)
    for _ in range(300):
        sc = xs ** 3 / y * w
        c, *_ = np.linalg.lstsq(A * sc[:, None], tgt * sc, rcond=None)
        err = (xs + xs ** 3 * (A @ c) - y) / y
        w = w * np.abs(err) ** 0.5
        w /= w.max()
    return c.astype(np.float32)


def evaluate(c, top=0.5):
    fma = lambda a, b, d: (a.astype(np.float64) * b + d).astype(np.float32)
    lo, hi = np.float32(2 ** -12).view(np.int32), np.float32(top).view(np.int32)
    x = np.arange(lo, hi, dtype=np.int32).view(np.float32)
    s = (x * x).astype(np.float32)
    p = np.full_like(x, c[-1])
    for k in range(len(c) - 2, -1, -1):
        p = fma(p, s, np.full_like(x, c[k]))
    y = fma((s * x).astype(np.float32), p, x)
    ref = np.tanh(x.astype(np.float64))
    return float((np.abs(y - ref) / ref).max()), float((np.abs(y - ref) / np.spacing(ref.astype(np.float32))).max())


if __name__ == "__main__":
    c = fit()
    print("coefficients c0..c3:", [repr(float(v)) for v in c])
    print("max rel err %.3g, max ulp %.3f" % evaluate(c))
