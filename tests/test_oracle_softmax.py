"""Pins of the oracle's Softmax: float64 exactness of Alg 1 / Alg B (PAPER.md
705-713 doubling identity; G4 exponent), the polynomial tables' accuracy,
and the encrypted toy Softmax against float64 Softmax within the north-star
tolerance 2^-15, with the op counts of Alg 2 (PAPER.md 891-896)."""
import math
import os

import numpy as np
import pytest
from numpy.polynomial import chebyshev as Ch

import workloads as W
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def softmax64(x):
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def alg1_float(x, k):
    """PAPER.md 776-787 in float64 with exact exp and inverse square root."""
    y = np.exp(x / 2.0 ** k)
    for _ in range(k):
        lam = (y * y).sum(-1, keepdims=True) ** -0.5
        z = lam * y
        y = z * z
    return y


def algB_float(x, k, exponent="G4"):
    """PAPER.md 168-181; exponent -1/2^j (G4) or the printed -2^-(j-1)."""
    y0 = np.exp(x / 2.0 ** k)
    y, lam = y0, np.ones_like(y0[..., :1])
    for j in range(1, k + 1):
        e = -(0.5 ** j) if exponent == "G4" else -(2.0 ** -(j - 1))
        lam = lam * (y * y).sum(-1, keepdims=True) ** e
        y = (lam * y0) ** (2 ** j)
    return y


@pytest.mark.parametrize("M,n,k", [(128, 256, 5), (256, 128, 6), (2, 16, 1), (256, 1024, 6)])
def test_alg1_and_algB_exact_in_float64(M, n, k):
    x = W.softmax_inputs(64, n, M, seed=M * 1000 + n)
    ref = softmax64(x)
    assert np.abs(alg1_float(x, k) - ref).max() < 1e-13
    assert np.abs(algB_float(x, k) - ref).max() < 1e-13


def square_normalize_float(x, k):
    """PAPER.md 757-765 (G26): y <- y^2 / sum y^2, k times, from exp(x/2^k)."""
    y = np.exp(x / 2.0 ** k)
    for _ in range(k):
        w = y * y
        y = w / w.sum(-1, keepdims=True)
    return y


@pytest.mark.parametrize("M,n,k", [(128, 256, 5), (4, 16, 2)])
def test_square_and_normalize_exact_in_float64(M, n, k):
    x = W.softmax_inputs(64, n, M, seed=M * 7 + n)
    assert np.abs(square_normalize_float(x, k) - softmax64(x)).max() < 1e-13


def test_algB_printed_exponent_is_wrong_G4():
    x = W.softmax_inputs(16, 256, 128, seed=9)
    assert np.abs(algB_float(x, 5, "printed") - softmax64(x)).max() > 1e-2


def test_lemma_cs_range():
    """PAPER.md 721-728: sum y^2 in [1/n, 1] for y = Softmax(x/2^j)."""
    x = W.softmax_inputs(200, 64, 128, seed=3)
    for j in range(6):
        s = (softmax64(x / 2 ** j) ** 2).sum(-1)
        assert (s >= 1 / 64 - 1e-15).all() and (s <= 1 + 1e-15).all()


def test_input_distribution():
    x = W.softmax_inputs(1000, 256, 128, seed=1)
    assert x.min() >= -128 and x.max() <= 0
    assert abs(x.mean() + 64) < 0.2 and abs(x.std() - 128 / 6) < 0.5


def test_theorem_k_golden():
    for line in open(os.path.join(GOLD, "softmax_k.txt")):
        if line.startswith("#") or not line.strip():
            continue
        M, n, k = map(int, line.split())
        assert math.ceil(math.log2(M) - math.log2(math.log(n))) == k


def test_poly_tables_accuracy(tables):
    """Each table polynomial meets its recorded error bound on a dense grid,
    independently of the Remez code: exp absolute; x^-p weighted |P x^p - 1|."""
    for name, t in tables.items():
        e = t["exp"]
        xs = np.linspace(e["a"], e["b"], 20001)
        k = t["config"]["k"]
        tpow = 3 if t["config"]["variant"] == "T3" else 2
        err = np.abs(Ch.chebval((2 * xs - e["a"] - e["b"]) / (e["b"] - e["a"]), e["coeffs"]) - np.exp(xs / tpow ** k))
        assert err.max() <= e["max_err"] * 1.05 + 1e-15
        assert len(e["coeffs"]) - 1 == t["config"]["deg_exp"]
        for j, p in enumerate(t["inv"], start=1):
            var = t["config"]["variant"]
            pw = 0.5 if var == "A" else 1.0 if var in ("S", "T3") else 0.5 ** j
            xs = np.linspace(p["a"], p["b"], 20001)
            v = Ch.chebval((2 * xs - p["a"] - p["b"]) / (p["b"] - p["a"]), p["coeffs"])
            werr = np.abs(v * xs ** pw - 1)
            assert werr.max() <= p["max_err"] * 1.05
        # the last step is precise (PAPER.md 535-538: 19.5-bit final square root)
        last = t["inv"][-1]
        if last.get("newton"):
            # G24: seed + Newton y <- y (3 - x y^2)/2 (PAPER.md 1313-1316), run
            # in float64 on the grid: quadratic convergence to >= 19.5 bits
            xs = np.linspace(last["a"], last["b"], 20001)
            y = Ch.chebval((2 * xs - last["a"] - last["b"]) / (last["b"] - last["a"]), last["coeffs"])
            e0 = np.abs(y * np.sqrt(xs) - 1).max()
            for _ in range(last["newton"]):
                e_prev = np.abs(y * np.sqrt(xs) - 1)
                y = y * (3 - xs * y * y) / 2
                # PAPER.md 1322-1324: |y_n sqrt(x) - 1| <= 7/4 |y_(n-1) sqrt(x) - 1|^2
                assert (np.abs(y * np.sqrt(xs) - 1) <= 1.75 * e_prev ** 2 + 1e-15).all()
            assert e0 > 2.0 ** -13 and np.abs(y * np.sqrt(xs) - 1).max() < 2.0 ** -19.5
        elif t["config"]["k"] > 1 or name.startswith("toy_n16_M2"):
            assert last["log2_err"] < -13


def _toy_run(tables, wl_name, m, L, variant, table):
    wl = dict(W.WORKLOADS["config1"])
    P = O.Params.from_preset(W.preset("TOY12" if table.endswith("k1_A") else "TOY12D"))
    tab = tables[table]
    n, M, k = wl["n"], tab["config"]["M"], tab["config"]["k"]
    K = O.Keys(P, W.derive_seed("keys", wl_name), 192, galois=O.softmax_rotation_galois(P, n, m))
    x = W.softmax_inputs(L, n, M, seed=W.derive_seed("x", wl_name))
    slots = O.pack(x, P.n // 2, m)
    top = P.n_q - 1
    sc = O.softmax_input_scale(P, tab["exp"], top)  # G28
    cts = [O.encrypt(P, K, P.encode(slots[c], scale=sc, level=top), top,
                     W.derive_seed("enc", wl_name), c) for c in range(m)]
    O.ledger_reset()
    out = O.softmax(P, K, cts, n, k, variant, tab["exp"], tab["inv"])
    led = O.ledger()
    dec = np.stack([O.decrypt_decode(P, K, c).real for c in out])
    return x, dec, led, P, out


@pytest.mark.parametrize("m,table", [(1, "toy_n16_M2_k1_A"), (2, "toy_n16_M4_k2_A"), (2, "toy_n16_M4_k2_B"),
                                     (2, "toy_n16_M4_k2_A_nt"), (2, "toy_n16_M4_k2_S")])
def test_oracle_toy_softmax_accuracy(tables, m, table):
    L = 100 if m == 1 else 256
    variant = tables[table]["config"]["variant"]
    x, dec, led, P, out = _toy_run(tables, "config1", m, L, variant, table)
    n, k = 16, tables[table]["config"]["k"]
    got = O.unpack(dec, L, n)
    err = np.abs(got - softmax64(x)).max()
    assert err < 2.0 ** -15, math.log2(err)
    nb = n // m
    # Alg 2: 2 log2(nb) rotations per aux call (PAPER.md 891-896 / G6)
    assert led["rot"] == k * 2 * int(math.log2(nb))
    if m == 1:
        # padding lanes carry x = 0 -> output 1/n (G9)
        stride = (P.n // 2) // nb
        pad = np.array([dec[0, b * stride + o] for b in range(nb) for o in range(L, stride)])
        assert np.abs(pad - 1 / n).max() < 2.0 ** -15


def test_oracle_newton_step_pin():
    """G24 / PAPER.md 1313-1327: one encrypted Newton step from x/2 and a seed
    y0 costs 2 levels and obeys |y1 sqrt(x) - 1| <= 7/4 |y0 sqrt(x) - 1|^2
    (+ CKKS noise), for seeds off by up to 30 %."""
    P = O.Params.from_preset(W.preset("TOY12"))
    K = O.Keys(P, 4242, 192)
    rng = np.random.default_rng(5)
    x = rng.uniform(0.05, 1.0, P.n // 2)
    e0 = rng.uniform(-0.3, 0.3, P.n // 2)
    y0 = (1 + e0) / np.sqrt(x)
    top = P.n_q - 1
    cx = O.encrypt(P, K, P.encode(x, scale=P.scale(top), level=top), top, 1, 0)
    cy = O.encrypt(P, K, P.encode(y0, scale=P.scale(top - 1), level=top - 1), top - 1, 1, 1)
    xh = O.op(P, K, "mult_const", cx, c=0.5, i=top - 1)
    y1 = O.newton_step(P, K, xh, cy)
    assert y1.level == top - 3
    got = O.decrypt_decode(P, K, y1).real
    e1 = np.abs(got * np.sqrt(x) - 1)
    assert (e1 <= 1.75 * e0 ** 2 + 2.0 ** -20).all()
    # and the step is not the identity: the error really shrank
    assert e1.max() < 0.5 * np.abs(e0).max()


def test_oracle_newton_needed_for_toy_accuracy(tables):
    """Without its Newton steps the degree-7 seed alone misses 2^-15: the
    Newton path (not the polynomial) carries the accuracy of the _nt table."""
    t = dict(tables["toy_n16_M4_k2_A_nt"])
    t["inv"] = [dict(p) for p in t["inv"]]
    t["inv"][-1].pop("newton")
    x, dec, led, P, out = _toy_run({"nt0": t}, "config1", 2, 256, "A", "nt0")
    err = np.abs(O.unpack(dec, 256, 16) - softmax64(x)).max()
    assert err > 2.0 ** -15


def test_oracle_rejects_newton_with_version_b(tables):
    """G24: Newton steps are defined for Alg 1's x^(-1/2) only; the oracle
    rejects them with version B (ORC_EINVAL), as the C ABI does (HS_EINVAL)."""
    t = dict(tables["toy_n16_M4_k2_B"])
    t["inv"] = [dict(p) for p in t["inv"]]
    t["inv"][-1]["newton"] = 2
    with pytest.raises(RuntimeError, match="rc=1"):
        _toy_run({"ntB": t}, "config1", 2, 256, "B", "ntB")


def cube_normalize_float(x, k):
    """PAPER.md 1645-1663 (G27), t = 3: y <- y^3 / sum y^3, k times, from exp(x/3^k)."""
    y = np.exp(x / 3.0 ** k)
    for _ in range(k):
        w = y ** 3
        y = w / w.sum(-1, keepdims=True)
    return y


@pytest.mark.parametrize("M,n,k", [(4, 4, 2), (128, 128, 4)])
def test_cube_and_normalize_exact_in_float64(M, n, k):
    x = W.softmax_inputs(64, n, M, seed=M + 3 * n)
    assert np.abs(cube_normalize_float(x, k) - softmax64(x)).max() < 1e-13


def cube_toy_run(tables):
    tab = tables["toy_n4_M4_k2_T3"]
    cfg = tab["config"]
    n, M, k, m = cfg["n"], cfg["M"], cfg["k"], 2
    P = O.Params.from_preset(W.preset("TOY12D"))
    K = O.Keys(P, W.derive_seed("keys", "cube"), 192, galois=O.softmax_rotation_galois(P, n, m))
    L = (P.n // 2) * m // n
    x = W.softmax_inputs(L, n, M, seed=W.derive_seed("x", "cube"))
    slots = O.pack(x, P.n // 2, m)
    top = P.n_q - 1
    sc = O.softmax_input_scale(P, tab["exp"], top)  # G28
    cts = [O.encrypt(P, K, P.encode(slots[c], scale=sc, level=top), top, 11, c) for c in range(m)]
    out = O.softmax(P, K, cts, n, k, "T3", tab["exp"], tab["inv"])
    dec = np.stack([O.decrypt_decode(P, K, c).real for c in out])
    return x, O.unpack(dec, L, n)


def test_oracle_cube_and_normalize_toy(tables):
    """G27 on the toy ring: encrypted cube-and-normalize within 2^-15."""
    x, y = cube_toy_run(tables)
    assert np.abs(y - softmax64(x)).max() < 2.0 ** -15
