"""Pins of the bootstrapping's linear transforms (G11; SURVEY 8(c)
G11 "CtS o StC = id in float64") against the mathematics, not the oracle's
own ciphertext path: the special-FFT stage groups the plan encodes, composed
in float64, must (1) compose to the canonical embedding of C4 -- slot j is the
evaluation at zeta^(5^j mod 2N), zeta = exp(i pi / N), of the complex
coefficient vector w_k = m_k + i m_{k+N0} in bit-reversed order, i.e.
z = E P w with E[j][k] = zeta^(5^j k) -- and (2) the CoeffToSlot groups,
applied largest stage first as the plan applies them, must invert the
SlotToCoeff groups: CtS o StC = id, for every grouping the presets use."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O


def group(log_n, first, size, inverse):
    n0 = 1 << (log_n - 1)
    L = O.lib()
    f = L.orc_api_sfft_group
    f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, np.ctypeslib.ndpointer(np.float64),
                  np.ctypeslib.ndpointer(np.float64)]
    re, im = np.zeros(n0 * n0), np.zeros(n0 * n0)
    f(log_n, first, size, 1 if inverse else 0, re, im)
    return (re + 1j * im).reshape(n0, n0)


def sizes(s, g):
    """the plan's grouping rule (earlier groups not smaller)"""
    out, rem = [], s
    for k in range(g, 0, -1):
        out.append(-(-rem // k))
        rem -= out[-1]
    return out


def brv(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


@pytest.mark.parametrize("log_n,n_stc,n_cts", [(5, 2, 2), (6, 3, 4), (7, 3, 4), (8, 4, 3)])
def test_stc_is_canonical_embedding_and_cts_inverts_it(log_n, n_stc, n_cts):
    N, n0 = 1 << log_n, 1 << (log_n - 1)
    s = log_n - 1
    # SlotToCoeff: groups in stage order, group 0 applied first
    stc = np.eye(n0, dtype=complex)
    first = 0
    for sz in sizes(s, n_stc):
        stc = group(log_n, first, sz, False) @ stc
        first += sz
    zeta = np.exp(1j * np.pi / N)
    E = np.array([[zeta ** ((pow(5, j, 2 * N) * k) % (2 * N)) for k in range(n0)] for j in range(n0)])
    Pm = np.zeros((n0, n0))
    for k in range(n0):
        Pm[k, brv(k, s)] = 1.0
    assert np.abs(stc - E @ Pm).max() < 1e-12
    # the embedding itself, against direct polynomial evaluation (C4)
    rng = np.random.default_rng(log_n)
    m = rng.normal(size=N)
    z_direct = np.array([np.polyval(m[::-1], zeta ** pow(5, j, 2 * N)) for j in range(n0)])
    w = m[:n0] + 1j * m[n0:]
    assert np.abs(E @ w - z_direct).max() < 1e-9
    # CoeffToSlot: inverse groups, the LAST stage group applied first
    cts = np.eye(n0, dtype=complex)
    sz = sizes(s, n_cts)
    firsts = np.cumsum([0] + sz[:-1])
    for gi in reversed(range(n_cts)):
        cts = group(log_n, int(firsts[gi]), sz[gi], True) @ cts
    assert np.abs(cts @ stc - np.eye(n0)).max() < 1e-12
    assert np.abs(stc @ cts - np.eye(n0)).max() < 1e-12


def test_cts_transforms_c17_apply_the_matrices():
    """C17 (double-hoisted BSGS) pinned against the mathematics: on the
    N = 2^12 ring with P16's chain, a ciphertext at the top level holding slot
    vector z is run through the oracle's bootstrap up to its s-th
    CoeffToSlot transform (orc_bts_debug_stop, ModRaise skipped); its
    decryption must be f (T_{s-1} ... T_0) z, where T_k are the float64
    stage-group matrices above and f = (Delta_L / q_0) / (2 (K + 2)) the
    first transform's factor, within CKKS noise."""
    import workloads as W
    pre = W.preset("TOY12B")
    P = O.Params.from_preset(pre)
    cfg = pre["bts"]
    tab = W.bts_tables()[cfg["table"]]
    rots = O.bts_rotations(P, cfg)
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    K = O.Keys(P, 4321, pre["h"], galois=gal)
    B = O.Bts(P, cfg, tab)
    L_top = P.n_q - 1
    n0, log_n = P.n // 2, P.log_n
    s = log_n - 1
    rng = np.random.default_rng(3)
    z = rng.uniform(-1, 1, n0)
    ct = O.encrypt(P, K, P.encode(z, scale=P.scale(L_top), level=L_top), L_top, 5, 0, use_sk=True)
    f = (P.scale(L_top) / P.primes[0]) / (2 * (tab["K"] + 2))
    sz = sizes(s, cfg["n_cts"])
    firsts = np.cumsum([0] + sz[:-1])
    L = O.lib()
    L.orc_api_bts_debug_stop.argtypes = [C.c_int]
    L.orc_api_bts_debug_skip_raise.argtypes = [C.c_int]
    M = np.eye(n0, dtype=complex)
    try:
        L.orc_api_bts_debug_skip_raise(1)
        for stop in range(1, cfg["n_cts"] + 1):
            gi = cfg["n_cts"] - stop
            M = group(log_n, int(firsts[gi]), sz[gi], True) @ M
            L.orc_api_bts_debug_stop(stop)
            out = O.bootstrap(P, K, ct, B, 1.0)
            assert out.level == L_top - stop
            got = O.decrypt_decode(P, K, out)
            want = f * (M @ z)
            err = np.abs(got - want).max() / np.abs(want).max()
            assert err < 2.0 ** -20, (stop, np.log2(err))
    finally:
        L.orc_api_bts_debug_stop(-1)
        L.orc_api_bts_debug_skip_raise(0)


def test_evalmod_c18_even_series():
    """C18 pinned: the oracle's EvalMod stage (the even cosine series
    evaluated as a half-degree series on w = T_2(v) = 2v^2 - 1) must decrypt
    to float64 Clenshaw of the FULL degree-63 table at the decrypted v
    (orc_bts_debug_stop 10 -> v, 11 -> the series), within CKKS noise."""
    from numpy.polynomial import chebyshev as Ch
    import workloads as W
    pre = W.preset("TOY12B")
    P = O.Params.from_preset(pre)
    cfg = pre["bts"]
    tab = W.bts_tables()[cfg["table"]]
    assert all(c == 0.0 for c in tab["coeffs"][1::2])  # even: the C18 case
    rots = O.bts_rotations(P, cfg)
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    K = O.Keys(P, 99, pre["h"], galois=gal)
    B = O.Bts(P, cfg, tab)
    L_top = P.n_q - 1
    z = np.random.default_rng(8).uniform(-1, 1, P.n // 2)
    ct = O.encrypt(P, K, P.encode(z, scale=P.scale(L_top), level=L_top), L_top, 5, 0, use_sk=True)
    L = O.lib()
    L.orc_api_bts_debug_stop.argtypes = [C.c_int]
    L.orc_api_bts_debug_skip_raise.argtypes = [C.c_int]
    try:
        L.orc_api_bts_debug_skip_raise(1)
        L.orc_api_bts_debug_stop(10)
        v = O.decrypt_decode(P, K, O.bootstrap(P, K, ct, B, 1.0)).real
        L.orc_api_bts_debug_stop(11)
        sct = O.bootstrap(P, K, ct, B, 1.0)
        got = O.decrypt_decode(P, K, sct).real
    finally:
        L.orc_api_bts_debug_stop(-1)
        L.orc_api_bts_debug_skip_raise(0)
    assert np.abs(v).max() <= 1.0
    want = Ch.chebval(v, tab["coeffs"])
    assert np.abs(got - want).max() < 2.0 ** -20, np.log2(np.abs(got - want).max())
