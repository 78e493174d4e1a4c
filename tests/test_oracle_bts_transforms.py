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
