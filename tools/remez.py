"""Offline weighted-minimax (Remez) generator for the Softmax polynomial tables.

PAPER.md 423-427 [sec 5.1.2]: the paper computed its approximants with Sollya:
minimax for exp, and for x^(-1/2) the *weighted* minimax that minimises
||P(x) sqrt(x) - 1||_inf; degrees of the form 2^t - 1.  The coefficients were
not printed (G15), so this tool recomputes them.  It is host tooling
that writes DATA (data/poly_tables.json); the tables are method parameters that
both the CUDA path and the oracle receive as inputs, like the paper's Sollya
output.  Neither side imports this module.

Representation: Chebyshev series on [a, b]: P(x) = sum_i c_i T_i(u),
u = (2x - a - b) / (b - a).

Usage:  python tools/remez.py [names...]  (rewrites data/poly_tables.json, or only the named tables)
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
from numpy.polynomial import chebyshev as Ch


def _cheb_vander(u, d):
    return Ch.chebvander(u, d)


def remez(f, w, a, b, d, iters=60, grid=None, tol=1e-3):
    """Weighted minimax: minimise max_x |w(x) (f(x) - P(x))| over [a, b].

    Returns (coeffs, max_weighted_error).  Classical multiple-exchange Remez in
    the Chebyshev basis, float64 (well conditioned up to degree ~255).
    """
    n_grid = grid or max(4000, 40 * (d + 2))
    # dense grid clustered at the end points (Chebyshev-Lobatto in u)
    ug = -np.cos(np.pi * np.arange(n_grid) / (n_grid - 1))
    xg = 0.5 * (b - a) * ug + 0.5 * (a + b)
    fg, wg = f(xg), w(xg)
    Vg = _cheb_vander(ug, d)
    # initial reference: Chebyshev extrema of T_{d+1}
    ref = np.sort(-np.cos(np.pi * np.arange(d + 2) / (d + 1)))
    best = None
    for _ in range(iters):
        xr = 0.5 * (b - a) * ref + 0.5 * (a + b)
        A = np.zeros((d + 2, d + 2))
        A[:, : d + 1] = _cheb_vander(ref, d)
        A[:, d + 1] = [(-1) ** i / w(np.array([x]))[0] for i, x in enumerate(xr)]
        sol = np.linalg.solve(A, f(xr))
        c = sol[: d + 1]
        err = wg * (fg - Vg @ c)
        emax = np.max(np.abs(err))
        if best is None or emax < best[1]:
            best = (c.copy(), emax)
        # new reference: extremum of each sign-constant run
        s = np.sign(err)
        s[s == 0] = 1
        runs, start = [], 0
        for i in range(1, n_grid + 1):
            if i == n_grid or s[i] != s[start]:
                j = start + int(np.argmax(np.abs(err[start:i])))
                runs.append(j)
                start = i
        # keep d+2 alternating points with the largest |err| (drop smallest
        # interior/end runs while too many)
        while len(runs) > d + 2:
            vals = [abs(err[j]) for j in runs]
            # remove the smaller of the two end points or the smallest pair
            if vals[0] < vals[-1]:
                runs.pop(0)
            else:
                runs.pop()
        if len(runs) < d + 2:
            break
        new_ref = ug[runs]
        levelled = (np.max(np.abs(err[runs])) - np.min(np.abs(err[runs]))) / emax
        ref = np.sort(new_ref)
        if levelled < tol:
            break
    return best


def cheb_eval(coeffs, a, b, x):
    u = (2 * np.asarray(x, dtype=np.float64) - a - b) / (b - a)
    return Ch.chebval(u, coeffs)


def make_exp(M, k, deg, t=2):
    f = lambda x: np.exp(x / float(t) ** k)
    c, e = remez(f, lambda x: np.ones_like(x), -float(M), 0.0, deg)
    return dict(func=f"exp(x/{t}^{k})", a=-float(M), b=0.0, coeffs=[float(v) for v in c], weight="abs",
                max_err=float(e), log2_err=float(math.log2(e)))


def make_invpow(p, a, b, deg):
    """Weighted minimax of x^(-p): minimise |P(x) x^p - 1| (PAPER.md 424)."""
    f = lambda x: x ** (-p)
    w = lambda x: x ** p
    c, e = remez(f, w, float(a), float(b), deg)
    return dict(func=f"x^(-{p})", a=float(a), b=float(b), coeffs=[float(v) for v in c], weight="rel",
                max_err=float(e), log2_err=float(math.log2(e)))


def softmax_tables(n, M, k, variant, deg_exp, deg_first, deg_mid, deg_last, guard=0.02, alpha=None, newton=0):
    if variant == "T3":
        return power_tables(n, M, k, 3, deg_exp, deg_first, deg_mid, deg_last, guard)
    """Per-iteration polynomial list for one (n, M, k, variant) configuration.

    First interval  [n e^{-M/2^(k-1)} (1-guard), n (1+guard)]   (PAPER.md 1001-1002)
    Later intervals [(1-alpha)^2/n, (1+alpha)^2]                  (PAPER.md 427)
    alpha = 2 * (weighted error of the previous step), i.e. |x P^2 - 1|.
    newton > 0 (Alg 1 only): the last polynomial is a minimax SEED followed by
    `newton` inverse-square-root Newton steps (PAPER.md 1311-1327 [App. A]:
    |y_n sqrt(x) - 1| <= 7/4 |y_(n-1) sqrt(x) - 1|^2), DESIGN.md G24.
    """
    polys = {"exp": make_exp(M, k, deg_exp)}
    lo = n * math.exp(-M / 2.0 ** (k - 1)) * (1 - guard)
    hi = n * (1 + guard)
    inv = []
    prev_alpha = None
    for j in range(1, k + 1):
        # Alg 1: x^-1/2; version B: x^-1/2^j (G4); square-and-normalize: x^-1 (G26)
        p = 0.5 if variant == "A" else 1.0 if variant == "S" else 0.5 ** j
        if j == 1:
            a, b = lo, hi
            deg = deg_first if k > 1 else deg_last
        else:
            al = prev_alpha * (1 + guard) + guard / 4
            a, b = (1 - al) ** 2 / n, (1 + al) ** 2
            deg = deg_last if j == k else deg_mid
        pol = make_invpow(p, a, b, deg)
        if j == k and newton:
            assert variant == "A"
            e = pol["max_err"]
            for _ in range(newton):
                e = 1.75 * e * e
            pol["newton"] = int(newton)
            pol["newton_log2_err_bound"] = float(math.log2(e))
        # |x P(x)^(1/p) - 1|: P ~ x^-p within relative e  ->  x P^(1/p) within ~ e/p
        prev_alpha = pol["max_err"] / p
        pol["alpha_out"] = prev_alpha
        inv.append(pol)
    polys["inv"] = inv
    return polys


def power_tables(n, M, k, t, deg_exp, deg_first, deg_mid, deg_last, guard=0.02):
    """t-th power normalization (PAPER.md 1645-1663 [App. C], G27): y0 =
    exp(x/t^k); mu_j = P_j(sum y^t) ~ (sum y^t)^-1 (weighted minimax of x^-1);
    first interval [n e^(-t M / t^k), n], then, with sum y within alpha of 1,
    [(1-alpha)^t / n^(t-1), (1+alpha)^t] (Hoelder)."""
    polys = {"exp": make_exp(M, k, deg_exp, t)}
    inv, prev_alpha = [], None
    for j in range(1, k + 1):
        if j == 1:
            a = n * math.exp(-t * M / float(t) ** k) * (1 - guard)
            b = n * (1 + guard)
            deg = deg_first if k > 1 else deg_last
        else:
            al = prev_alpha * (1 + guard) + guard / 4
            a, b = (1 - al) ** t / n ** (t - 1), (1 + al) ** t
            deg = deg_last if j == k else deg_mid
        pol = make_invpow(1.0, a, b, deg)
        prev_alpha = pol["max_err"]
        pol["alpha_out"] = prev_alpha
        inv.append(pol)
    polys["inv"] = inv
    return polys


CONFIGS = {
    # config 1 (TOY12): n = 16, M = 2, k = 1 (forced), Alg 1
    "toy_n16_M2_k1_A": dict(n=16, M=2, k=1, variant="A", deg_exp=7, deg_first=15, deg_mid=15, deg_last=15),
    # toy with two iterations (exercises first/last split) -- parity only
    "toy_n16_M4_k2_A": dict(n=16, M=4, k=2, variant="A", deg_exp=7, deg_first=7, deg_mid=7, deg_last=31),
    "toy_n16_M4_k2_B": dict(n=16, M=4, k=2, variant="B", deg_exp=7, deg_first=7, deg_mid=7, deg_last=31),
    # Newton variant of the k = 2 toy: degree-7 seed + 2 Newton steps (G24) -- pins only
    "toy_n16_M4_k2_A_nt": dict(n=16, M=4, k=2, variant="A", deg_exp=7, deg_first=7, deg_mid=7, deg_last=7,
                               newton=2),
    # square-and-normalize (PAPER.md 757-765, G26) at the k = 2 toy shape
    "toy_n16_M4_k2_S": dict(n=16, M=4, k=2, variant="S", deg_exp=7, deg_first=15, deg_mid=15, deg_last=31),
    # cube-and-normalize (t = 3, App. C, G27) at the toy shape: x/3^k, k = 2
    "toy_n4_M4_k2_T3": dict(n=4, M=4, k=2, variant="T3", deg_exp=7, deg_first=15, deg_mid=31, deg_last=31),
    # P16 configs 2-4 (n=256/128, M=128, k=5)
    "p16_n256_M128_k5_A": dict(n=256, M=128, k=5, variant="A", deg_exp=15, deg_first=63, deg_mid=31, deg_last=127),
    # version B (configs 3, 4): exp degree 11 -- the same 4 levels as degree 15
    # (tab:depth_main), 2^-31 absolute instead of 2^-45 (below the CKKS noise
    # floor either way), and 6 instead of 8 products on every one of the m
    # main-thread ciphertexts (G30)
    "p16_n256_M128_k5_B": dict(n=256, M=128, k=5, variant="B", deg_exp=11, deg_first=63, deg_mid=31, deg_last=127),
    "p16_n128_M128_k5_B": dict(n=128, M=128, k=5, variant="B", deg_exp=11, deg_first=63, deg_mid=31, deg_last=127),
    # config 2 with square-and-normalize (G26): x^-1 needs degree 63 where x^-1/2 takes 31
    "p16_n256_M128_k5_S": dict(n=256, M=128, k=5, variant="S", deg_exp=15, deg_first=63, deg_mid=63, deg_last=127),
    # config 5 (n = N0 = 32768, M = 256, Alg 1, k = 7): degree-255
    # middle steps, last step = degree-255 seed + 3 Newton steps (G24)
    "p16_n32768_M256_k7_A": dict(n=32768, M=256, k=7, variant="A", deg_exp=15, deg_first=15, deg_mid=255,
                                 deg_last=255, newton=3),
    # the config-5 schedule at n = N0 of the N = 2^12 ring (TOY12B): parity only
    # (degree 63 at n = 2048 ~ degree 255 at n = 32768: the seed needs the Newton steps)
    "toy_n2048_M32_k4_A": dict(n=2048, M=32, k=4, variant="A", deg_exp=15, deg_first=15, deg_mid=63,
                               deg_last=63, newton=3),
}


def main(out_path=None, only=None):
    """only: names to (re)compute; the other tables already in out_path are kept."""
    out_path = out_path or os.path.join(os.path.dirname(__file__), "..", "data", "poly_tables.json")
    tables = {}
    if only and os.path.exists(out_path):
        with open(out_path) as fh:
            tables = json.load(fh)
    for name, cfg in CONFIGS.items():
        if only and name not in only:
            continue
        t = softmax_tables(**cfg)
        t["config"] = cfg
        tables[name] = t
        print(name, "exp", round(t["exp"]["log2_err"], 1),
              "inv", [round(p["log2_err"], 1) for p in t["inv"]], file=sys.stderr)
    with open(out_path, "w") as fh:
        json.dump(tables, fh, indent=1)
    return tables


if __name__ == "__main__":
    main(only=sys.argv[1:] or None)
