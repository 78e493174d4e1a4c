"""Offline generator of the bootstrapping EvalMod polynomial (data/bts_tables.json).

EvalMod (reading G11) evaluates, on v in [-1, 1],
    g(v) = cos(2 pi (K + 2) v / 2^r)
followed by r double-angle steps, so that cos(2 pi (y - 1/4)) = sin(2 pi y) for
v = (y - 1/4) / (K + 2).  The Chebyshev coefficients of g are exact
(Jacobi-Anger): cos(w t) = J_0(w) + 2 sum_{k>=1} (-1)^k J_{2k}(w) T_{2k}(t),
truncated at the table degree; computed with mpmath at 50 digits.  Like the
Softmax tables this is DATA that both the CUDA path and the oracle receive.
"""
import json
import os

import mpmath as mp

mp.mp.dps = 50


def cos_table(K, r, deg):
    w = 2 * mp.pi * (K + 2) / mp.mpf(2) ** r
    c = [mp.mpf(0)] * (deg + 1)
    c[0] = mp.besselj(0, w)
    for k in range(1, deg // 2 + 1):
        c[2 * k] = 2 * (-1) ** k * mp.besselj(2 * k, w)
    tail = sum(abs(2 * mp.besselj(2 * k, w)) for k in range(deg // 2 + 1, deg // 2 + 40))
    return dict(K=K, r=r, deg=deg, a=-1.0, b=1.0, coeffs=[float(x) for x in c], trunc_err=float(tail))


def main():
    # (K, r, deg): EvalMod depth = cheb_depth(deg) + r; K24_r4_d31 has the same
    # depth as K24_r3_d63 (6 + 4 = 7 + 3) with 4 fewer ciphertext products
    specs = [(24, 3, 63), (12, 3, 63), (24, 2, 127), (24, 1, 255), (24, 4, 63), (24, 3, 31), (24, 4, 31)]
    out = {f"K{K}_r{r}_d{d}": cos_table(K, r, d) for K, r, d in specs}
    path = os.path.join(os.path.dirname(__file__), "..", "data", "bts_tables.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    for k, v in out.items():
        print(k, "truncation error", v["trunc_err"])


if __name__ == "__main__":
    main()
