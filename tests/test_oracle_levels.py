"""Level budget of the oracle pinned to the paper's printed depth tables
(tests/golden/depth_tables.txt): PAPER.md 330-336 (ceil(log(d+1)) levels for a
degree-d polynomial), tab:depth_main (PAPER.md 964-979: exp depth 4, main
thread 2k + 4) and tab:depth_aux_thread (PAPER.md 1032-1058, n = 256: square
and mask 2, x^(-1/2) depths 6, 5 x (k-2), 7).

The runs use a deep test-only chain at N = 2^10 (insecure, no bootstrapping)
so that every step's level drop is visible in the oracle's level trace; the
decrypted outputs are also checked against float64, so a schedule that saved
levels by computing something else would fail."""
import math
import os

import numpy as np
import pytest
from numpy.polynomial import chebyshev as Ch

import workloads as W
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "depth_tables.txt")


def gold():
    out = {}
    for line in open(GOLD):
        if line.strip() and not line.startswith("#"):
            k, v = line.split()
            out[k] = int(v)
    return out


def deep_params(n_levels):
    """N = 2^10, q0 60 bits + n_levels user primes of 40 bits (Delta = 2^40), 8
    special primes (alpha = 8): deep enough to run a whole Softmax unbootstrapped."""
    q = [60] + [40] * n_levels
    anchors = [0] * len(q)
    anchors[-1] = 40
    return O.Params(10, q, [61] * 8, 8, anchors)


def softmax64(x):
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


@pytest.fixture(scope="module")
def deep():
    P = deep_params(52)
    gal = set(O.softmax_rotation_galois(P, 256, 1))
    K = O.Keys(P, 2024, 64, galois=sorted(gal))
    return P, K


@pytest.mark.parametrize("which", ["exp", 0, 1, 4])
def test_config3_polynomial_depths(deep, tables, which):
    """Each polynomial of the config-3 table consumes exactly the levels the
    paper prints for n = 256: exp 4; x^(-1/2^j) 6 (first), 5 (middle), 7
    (last) -- i.e. ceil(log2(d+1)) for the degrees 15 / 63 / 31 / 127 -- and
    evaluates to float64 Clenshaw of the same series."""
    G = gold()
    P, K = deep
    tab = tables["p16_n256_M128_k5_B"]
    p = tab["exp"] if which == "exp" else tab["inv"][which]
    want = {"exp": G["main_exp_depth"], 0: G["aux_inv_first_n256"], 1: G["aux_inv_middle_n256"],
            4: G["aux_inv_last_n256"]}[which]
    deg = len(p["coeffs"]) - 1
    assert want == math.ceil(math.log2(deg + 1))
    rng = np.random.default_rng(7)
    x = rng.uniform(p["a"], p["b"], P.n // 2)
    top = P.n_q - 1
    ct = O.encrypt(P, K, P.encode(x, scale=P.scale(top) * 2.0 / (p["b"] - p["a"]), level=top), top, 3, 0)
    out = O.cheb(P, K, ct, p)
    assert top - out.level == want
    ref = Ch.chebval((2 * x - p["a"] - p["b"]) / (p["b"] - p["a"]), p["coeffs"])
    got = O.decrypt_decode(P, K, out).real
    assert np.abs(got - ref).max() < 2.0 ** -20 * max(1.0, np.abs(ref).max())


def run_traced(P, K, table, variant, n, m, L, M):
    k = table["config"]["k"] if "k" in table["config"] else len(table["inv"])
    x = W.softmax_inputs(L, n, M, seed=W.derive_seed("x", "levels", n))
    slots = O.pack(x, P.n // 2, m)
    top = P.n_q - 1
    sc = O.softmax_input_scale(P, table["exp"], top)
    cts = [O.encrypt(P, K, P.encode(slots[c], scale=sc, level=top), top, 5, c) for c in range(m)]
    O.trace(True)
    out = O.softmax(P, K, cts, n, k, variant, table["exp"], table["inv"])
    tr = O.trace_get()
    O.trace(False)
    dec = np.stack([O.decrypt_decode(P, K, c).real for c in out])
    err = np.abs(O.unpack(dec, L, n) - softmax64(x)).max()
    return tr, err, k


def test_alg1_level_budget_matches_paper(deep, tables):
    """Alg 1 on the config-2 table (n = 256, M = 128, k = 5), unbootstrapped:
    exp 4; per iteration the aux thread spends square 1 + x^(-1/2) (6, 5, 5, 5,
    7) + mask 1 (tab:depth_aux_thread: 2 + d_inv), the main thread 2
    (tab:depth_main: 2k + 4 in total); the output is Softmax within 2^-15."""
    G = gold()
    P, K = deep
    tab = tables["p16_n256_M128_k5_A"]
    tr, err, k = run_traced(P, K, tab, "A", 256, 1, 2, 128.0)
    ev = lambda name: [t for t in tr if t[0] == name]
    (e,) = ev("exp")
    assert e[2] - e[3] == G["main_exp_depth"]
    inv = [G["aux_inv_first_n256"]] + [G["aux_inv_middle_n256"]] * (k - 2) + [G["aux_inv_last_n256"]]
    assert [a - b for _, _, a, b in ev("poly")] == inv
    sq = [a - b for _, _, a, b in ev("square")]
    mk = [a - b for _, _, a, b in ev("mask")]
    assert [s + m_ for s, m_ in zip(sq, mk)] == [G["aux_sq_mask"]] * k
    main = [a - b for _, _, a, b in ev("main")]
    assert main == [G["main_per_iteration"]] * k
    assert G["main_exp_depth"] + sum(main) == 2 * k + 4  # tab:depth_main
    assert not ev("bts_main") and not ev("bts_aux")
    assert err < 2.0 ** -15, math.log2(err)


def test_algB_main_thread_depth(tables):
    """Version B (Alg B, PAPER.md 168-181; toy k = 2 table), unbootstrapped:
    the main update of iteration j reads lambda and y0 and spends 1 + j levels
    (z = lambda y0, then j squarings); exp 3 for degree 7; the aux polynomials
    ceil(log2(d+1)) = 3 and 5; the output within 2^-15 of float64 Softmax."""
    G = gold()
    P = deep_params(30)
    tab = tables["toy_n16_M4_k2_B"]
    n, m = 16, 2
    K = O.Keys(P, 77, 64, galois=O.softmax_rotation_galois(P, n, m))
    tr, err, k = run_traced(P, K, tab, "B", n, m, (P.n // 2) * m // n, 4.0)
    main = [(j, a - b) for ev, j, a, b in tr if ev == "main"]
    assert main == [(j, G["algB_main_iteration_extra"] + j) for j in range(1, k + 1)]
    assert [a - b for ev, _, a, b in tr if ev == "poly"] == [3, 5]
    (e,) = [t for t in tr if t[0] == "exp"]
    assert e[2] - e[3] == 3
    assert err < 2.0 ** -15, math.log2(err)
