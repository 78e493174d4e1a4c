"""Pins of the oracle's CKKS layer: exact big-integer identities on a tiny ring
(rescale C9, key switching C7, tensor C8) and homomorphism within noise bounds
(PAPER.md 298-304: ||Dec(op(ct)) - op(Dec ct)||_inf small; op precision
~29 bits, PAPER.md 388-389)."""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from tests import refmath as R


@pytest.fixture(scope="module")
def tiny():
    P = O.Params.from_preset(W.preset("TINY"))
    K = O.Keys(P, 21, 8, galois=[P.galois_of_rot(1), 2 * P.n - 1], relin=True)
    return P, K


@pytest.fixture(scope="module")
def toy():
    P = O.Params.from_preset(W.preset("TOY12"))
    gal = sorted({P.galois_of_rot(r) for r in [1, -1, 3, 128, -128, 256]} | {2 * P.n - 1})
    K = O.Keys(P, 77, 192, galois=gal, relin=True)
    return P, K


def coeff_ints(P, limbs, level):
    """NTT-domain limbs -> centred integers mod Q_level via the C3 definition + CRT."""
    cols = [R.intt_def([int(v) for v in limbs[i]], P.primes[i], P.psi(i), P.log_n) for i in range(level + 1)]
    out = []
    for t in range(P.n):
        x, Q = R.crt([cols[i][t] for i in range(level + 1)], P.primes[: level + 1])
        out.append(R.centred(x, Q))
    return out, Q


def enc(P, K, z, level, idx=0, sk=True):
    pt = P.encode(np.real(z), np.imag(z) if np.iscomplexobj(z) else None, scale=P.scale(level), level=level)
    return O.encrypt(P, K, pt, level, 1000 + idx, idx, use_sk=sk)


def test_rescale_is_rounded_division_C9(tiny):
    P, K = tiny
    rng = np.random.default_rng(0)
    ct = enc(P, K, rng.uniform(-1, 1, P.n // 2), 3)
    r = O.op(P, K, "rescale", ct)
    assert r.level == 2
    w, wr = ct.words(), r.words()
    ql = P.primes[3]
    for comp in range(2):
        a, _ = coeff_ints(P, w[comp], 3)
        b, Q2 = coeff_ints(P, wr[comp], 2)
        for t in range(P.n):
            # round(a/ql): a/ql is never a tie (ql odd); Python // floors
            expect = (2 * a[t] + ql) // (2 * ql)
            assert (b[t] - expect) % Q2 == 0


def test_keyswitch_identity_C7(tiny):
    """c0' + c1' s == d s^2 + e_ks (mod Q_l) with small e_ks, in big integers."""
    P, K = tiny
    rng = np.random.default_rng(1)
    s = [int(v) for v in K.secret()]
    s2 = R.negacyclic_mul(s, s)
    for level in [3, 1]:
        d = np.stack([rng.integers(0, P.primes[i], P.n, dtype=np.uint64) for i in range(level + 1)])
        o0, o1 = O.keyswitch(P, K, 0, level, d)
        D, Q = coeff_ints(P, d, level)
        A0, _ = coeff_ints(P, o0, level)
        A1, _ = coeff_ints(P, o1, level)
        lhs = [x + y for x, y in zip(A0, R.negacyclic_mul(A1, s))]
        rhs = R.negacyclic_mul(D, s2)
        err = [R.centred((x - y) % Q, Q) for x, y in zip(lhs, rhs)]
        assert max(abs(e) for e in err) < 2 ** 20, max(abs(e) for e in err)


def _auto(a, k, N):
    """X -> X^k on a coefficient list (negacyclic: X^N = -1)."""
    out = [0] * N
    for i, v in enumerate(a):
        e = (i * k) % (2 * N)
        if e < N:
            out[e] += v
        else:
            out[e - N] -= v
    return out


def test_hoisted_rotation_identity_C16(tiny):
    """C16 hoisting: (c0', c1') from ONE ModUp satisfies
    c0' + c1' s == sigma(c0 + c1 s) + e_ks (mod Q_l), small e_ks, in big integers,
    for every rotation served by the shared ModUp (here r = 1 twice: the
    second use must see the ModUp unchanged)."""
    P, K = tiny
    rng = np.random.default_rng(11)
    ct = enc(P, K, rng.uniform(-1, 1, P.n // 2), 3)
    outs = O.rotate_hoisted(P, K, ct, [1, 1])
    assert outs[0].words().tobytes() == outs[1].words().tobytes()
    s = [int(v) for v in K.secret()]
    k = P.galois_of_rot(1)
    w = ct.words()
    c0, Q = coeff_ints(P, w[0], 3)
    c1, _ = coeff_ints(P, w[1], 3)
    ph = [x + y for x, y in zip(c0, R.negacyclic_mul(c1, s))]
    want = _auto(ph, k, P.n)
    o = outs[0].words()
    d0, _ = coeff_ints(P, o[0], 3)
    d1, _ = coeff_ints(P, o[1], 3)
    got = [x + y for x, y in zip(d0, R.negacyclic_mul(d1, s))]
    err = [R.centred((x - y) % Q, Q) for x, y in zip(got, want)]
    assert max(abs(e) for e in err) < 2 ** 20, max(abs(e) for e in err)


def test_hoisted_rotations_decrypt_C16(toy):
    P, K = toy
    rng = np.random.default_rng(12)
    z = rng.uniform(-1, 1, P.n // 2)
    a = enc(P, K, z, 11, 0, sk=False)
    rots = [1, 3, -128, 256]
    outs = O.rotate_hoisted(P, K, a, rots)
    for r, c in zip(rots, outs):
        assert c.level == 11
        assert np.abs(O.decrypt_decode(P, K, c).real - np.roll(z, -r)).max() < 2.0 ** -22
    # hoisting changes the words (BConv vs sigma's sign flips) but not the message
    plain = O.op(P, K, "rotate", a, i=3)
    assert plain.words().tobytes() != outs[1].words().tobytes()


def test_fused_relin_rescale_identity_C8(tiny):
    """C8 HMult = tensor then ONE division of (P d + sum ModUp(d2) evk) by P q_l:
    c0' + c1' s == round((d0 + d1 s + d2 s^2) / q_l) + small, in big integers."""
    P, K = tiny
    rng = np.random.default_rng(13)
    a = enc(P, K, rng.uniform(-1, 1, P.n // 2), 3, 0)
    b = enc(P, K, rng.uniform(-1, 1, P.n // 2), 3, 1)
    d = O.op(P, K, "tensor", a, b)
    m = O.op(P, K, "mult", a, b)
    assert m.level == 2
    s = [int(v) for v in K.secret()]
    ints = lambda c, k, lv: coeff_ints(P, c.words()[k], lv)[0]
    Q3 = coeff_ints(P, d.words()[0], 3)[1]
    D = [x + y + z for x, y, z in zip(ints(d, 0, 3), R.negacyclic_mul(ints(d, 1, 3), s),
                                      R.negacyclic_mul(R.negacyclic_mul(ints(d, 2, 3), s), s))]
    D = [R.centred(v % Q3, Q3) for v in D]
    ql = P.primes[3]
    Q2 = coeff_ints(P, m.words()[0], 2)[1]
    M = [x + y for x, y in zip(ints(m, 0, 2), R.negacyclic_mul(ints(m, 1, 2), s))]
    err = [R.centred((mv - (2 * dv + ql) // (2 * ql)) % Q2, Q2) for mv, dv in zip(M, D)]
    # exact centred rounding (C7): only the two output roundings (|r0 + r1 s|
    # <= (1 + h)/2 = 4.5 for h = 8) plus the key-switch noise / (P q_l) < 1
    assert max(abs(e) for e in err) <= 6, max(abs(e) for e in err)


def test_tensor_identity_C8(tiny):
    """(d0 + d1 s + d2 s^2) == (a0 + a1 s)(b0 + b1 s) exactly mod Q_l."""
    P, K = tiny
    rng = np.random.default_rng(2)
    a = enc(P, K, rng.uniform(-1, 1, P.n // 2), 3, 0)
    b = enc(P, K, rng.uniform(-1, 1, P.n // 2), 3, 1)
    d = O.op(P, K, "tensor", a, b)
    s = [int(v) for v in K.secret()]
    ints = lambda c, k: coeff_ints(P, c.words()[k], 3)[0]
    Q = coeff_ints(P, a.words()[0], 3)[1]
    lhs = [x + y + z for x, y, z in zip(ints(d, 0), R.negacyclic_mul(ints(d, 1), s),
                                        R.negacyclic_mul(R.negacyclic_mul(ints(d, 2), s), s))]
    pa = [x + y for x, y in zip(ints(a, 0), R.negacyclic_mul(ints(a, 1), s))]
    pb = [x + y for x, y in zip(ints(b, 0), R.negacyclic_mul(ints(b, 1), s))]
    rhs = R.negacyclic_mul(pa, pb)
    assert all((x - y) % Q == 0 for x, y in zip(lhs, rhs))


def test_key_structure(tiny):
    """evk_j mod q_i = -a s + e + [i in D_j] P s^2 (checked as a small error)."""
    P, K = tiny
    k = K.swk(0)
    s = [int(v) for v in K.secret()]
    s2 = R.negacyclic_mul(s, s)
    Pm = 1
    for p in P.primes[P.n_q:]:
        Pm *= p
    for j in range(P.dnum):
        for i in range(P.n_q + P.n_p):
            q = P.primes[i]
            k0 = R.intt_def([int(v) for v in k[j, 0, i]], q, P.psi(i), P.log_n)
            k1 = R.intt_def([int(v) for v in k[j, 1, i]], q, P.psi(i), P.log_n)
            a_s = R.negacyclic_mul(k1, s, q)
            gadget = (Pm % q) if (i < P.n_q and i // P.alpha == j) else 0
            e = [R.centred((x + y - gadget * z) % q, q) for x, y, z in zip(k0, a_s, s2)]
            assert max(abs(v) for v in e) <= 21


def test_secret_is_sparse_ternary(toy):
    P, K = toy
    s = K.secret()
    assert set(np.unique(s)) <= {-1, 0, 1}
    assert int(np.count_nonzero(s)) == 192


def test_homomorphic_ops_within_noise(toy):
    P, K = toy
    rng = np.random.default_rng(3)
    za, zb = rng.uniform(-1, 1, P.n // 2), rng.uniform(-1, 1, P.n // 2)
    a, b = enc(P, K, za, 11, 0, sk=False), enc(P, K, zb, 8, 1, sk=False)
    dd = lambda c: O.decrypt_decode(P, K, c)
    tol = 2.0 ** -22
    assert np.abs(dd(a).real - za).max() < tol
    s = O.op(P, K, "add", a, b)
    assert s.level == 8 and np.abs(dd(s).real - (za + zb)).max() < tol
    m = O.op(P, K, "mult", a, b)
    assert m.level == 7 and np.abs(dd(m).real - za * zb).max() < tol
    r = O.op(P, K, "rotate", a, i=3)
    assert np.abs(dd(r).real - np.roll(za, -3)).max() < tol
    r = O.op(P, K, "rotate", a, i=-128)
    assert np.abs(dd(r).real - np.roll(za, 128)).max() < tol
    zc = za + 1j * zb
    c = O.op(P, K, "conj", enc(P, K, zc, 6, 2))
    assert np.abs(dd(c) - np.conj(zc)).max() < tol
    cm = O.op(P, K, "mult_const", a, c=-0.37, i=5)
    assert cm.level == 5 and np.abs(dd(cm).real + 0.37 * za).max() < tol
    ca = O.op(P, K, "add_const", a, c=0.25)
    assert np.abs(dd(ca).real - za - 0.25).max() < tol
    ld = O.op(P, K, "level_down", a, i=4)
    assert ld.level == 4 and np.abs(dd(ld).real - za).max() < tol
    mi = O.op(P, K, "mult_int", a, i=3)
    assert np.abs(dd(mi).real - 3 * za).max() < 3 * tol
    mask = (np.arange(P.n // 2) % 7 == 0).astype(float)
    pm = O.mult_pt(P, a, mask)
    assert pm.level == 10 and np.abs(dd(pm).real - za * mask).max() < tol


def test_canonical_scale_recurrence_C12():
    pre = W.preset("P16")
    P = O.Params.from_preset(pre)
    for lvl in range(len(pre["q_bits"])):
        if pre["log2_anchor"][lvl]:
            assert P.scale(lvl) == 2.0 ** pre["log2_anchor"][lvl]
        else:
            s = P.scale(lvl + 1)
            assert P.scale(lvl) == (s * s) / float(P.primes[lvl + 1])
    # user levels stay within 2^-16 of the anchored user scale (2^42)
    top_user = pre["bts"]["out_level"]
    assert all(abs(P.scale(l) / 2.0 ** pre["log2_anchor"][top_user] - 1) < 2.0 ** -16 for l in range(top_user + 1))


@pytest.mark.parametrize("deg,a,b,gain", [(7, -2.0, 0.0, 1.0), (15, 2.0, 16.5, 0.3), (31, -1.0, 1.0, 1.0),
                                          (2, 0.5, 3.0, 1.0), (1, 0.0, 4.0, 2.5), (63, -1.0, 1.0, 1.0),
                                          (5, -3.0, 1.0, 1.0), (8, 0.0, 2.0, 1.0)])
def test_chebyshev_eval_C13(toy, deg, a, b, gain):
    """Dec(eval(ct)) == gain * float64 Clenshaw of the same coefficients, and the
    evaluation consumes exactly ceil(log2(deg+1)) levels (PAPER.md 330-336:
    "a polynomial of degree d ... using ceil(log(d+1)) multiplicative levels";
    424-425: degree 2^t - 1 for a budget of t).  The input ciphertext holds
    alpha x, alpha = 2/(b-a) (x encoded at scale Delta alpha, G28)."""
    from numpy.polynomial import chebyshev as Ch
    P, K = toy
    rng = np.random.default_rng(deg)
    coeffs = rng.normal(0, 1, deg + 1) / (1 + np.arange(deg + 1)) ** 2
    z = rng.uniform(a, b, P.n // 2)
    top = P.n_q - 1
    pt = P.encode(z, scale=P.scale(top) * 2.0 / (b - a), level=top)
    ct = O.encrypt(P, K, pt, top, 1005, 5, use_sk=True)
    out = O.cheb(P, K, ct, dict(a=a, b=b, coeffs=coeffs), gain)
    t = max(1, int(np.ceil(np.log2(deg + 1))))
    assert out.level == top - t
    assert O.cheb_depth(deg) == t
    ref = gain * Ch.chebval((2 * z - a - b) / (b - a), coeffs)
    assert np.abs(O.decrypt_decode(P, K, out).real - ref).max() < 2.0 ** -20
