"""Pins of the oracle's ring layer against definitions it does not use itself:
Python big-integer prime search, the C3 NTT definition, schoolbook negacyclic
convolution, the coefficient-domain automorphism, RFC 8439's ChaCha20 vector,
Python's exact round-half-even, and a 50-digit mpmath encoding."""
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from tests import refmath as R

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def tiny():
    return O.Params.from_preset(W.preset("TINY"))


def _c1_primes(pre):
    """Independent recomputation of convention C1 (sized + derived primes)."""
    two_n = 2 << pre["log_n"]
    qb, pb, anc = pre["q_bits"], pre["p_bits"], pre["log2_anchor"]
    nq = len(qb)
    primes, taken = [None] * (nq + len(pb)), []

    def sized(bits):
        t = 1
        while True:
            q = (1 << bits) - t * two_n + 1
            if R.is_prime(q) and q not in taken:
                return q
            t += 1

    derived = [i >= 1 and anc[i - 1] == 0 for i in range(nq)]
    for i in range(nq):
        if not derived[i]:
            primes[i] = sized(qb[i]); taken.append(primes[i])
    for k, b in enumerate(pb):
        primes[nq + k] = sized(b); taken.append(primes[nq + k])
    scale = [0.0] * nq
    for l in range(nq - 1, -1, -1):
        scale[l] = 2.0 ** anc[l] if anc[l] else (scale[l + 1] * scale[l + 1]) / float(primes[l + 1])
        if l >= 1 and derived[l]:
            D = int(round(scale[l]))  # scale < 2^63, exact integer after rounding
            cands = []
            base = ((D - 1) // two_n) * two_n + 1
            for j in range(0, 4000):
                cands += [base - j * two_n, base + (j + 1) * two_n]
            cands.sort(key=lambda p: (abs(p - D), p))
            primes[l] = next(p for p in cands if R.is_prime(p) and p not in taken)
            taken.append(primes[l])
    return primes, scale


@pytest.mark.parametrize("name", ["TINY", "TOY12", "TOY12D", "P16"])
def test_prime_search_C1(name):
    pre = W.preset(name)
    P = O.Params.from_preset(pre)
    primes, scale = _c1_primes(pre)
    assert P.primes == primes
    assert [P.scale(l) for l in range(len(pre["q_bits"]))] == scale
    two_n = 2 << pre["log_n"]
    assert all(q % two_n == 1 for q in P.primes)
    assert len(set(P.primes)) == len(P.primes)
    assert all(q < 2 ** 60 for q in P.primes[: len(pre["q_bits"])])
    assert all(q < 2 ** 61 for q in P.primes)
    # derived primes keep the canonical scales stable (within 2^-16 of the anchor)
    for l, a in enumerate(pre["log2_anchor"]):
        if not a and l + 1 < len(pre["q_bits"]):
            up = next(x for x in pre["log2_anchor"][l + 1:] if x)
            assert abs(P.scale(l) / 2.0 ** up - 1) < 2.0 ** -16 or l == 0


@pytest.mark.parametrize("name", ["TINY", "TOY12"])
def test_psi_C2(name):
    pre = W.preset(name)
    P = O.Params.from_preset(pre)
    n = 1 << pre["log_n"]
    for i, q in enumerate(P.primes):
        psi = P.psi(i)
        assert pow(psi, n, q) == q - 1 and pow(psi, 2 * n, q) == 1
        x = 2
        while pow(pow(x, (q - 1) // (2 * n), q), n, q) != q - 1:
            x += 1
        assert psi == pow(x, (q - 1) // (2 * n), q)


def test_ntt_matches_definition_C3(tiny):
    rng = np.random.default_rng(0)
    for pi, q in enumerate(tiny.primes):
        a = [int(v) for v in rng.integers(0, q, tiny.n, dtype=np.uint64)]
        ref = R.ntt_def(a, q, tiny.psi(pi), tiny.log_n)
        assert [int(v) for v in tiny.ntt(pi, a)] == ref
        assert [int(v) for v in tiny.ntt_naive(pi, a)] == ref
        assert [int(v) for v in tiny.ntt(pi, ref, inverse=True)] == a


def test_ntt_larger_vs_naive():
    P = O.Params(log_n=10, q_bits=[60, 45], p_bits=[61], alpha=1, log2_anchor=[0, 40])
    rng = np.random.default_rng(1)
    for pi, q in enumerate(P.primes):
        a = rng.integers(0, q, P.n, dtype=np.uint64)
        assert (P.ntt(pi, a) == P.ntt_naive(pi, a)).all()


def test_negacyclic_convolution(tiny):
    rng = np.random.default_rng(2)
    for pi, q in enumerate(tiny.primes):
        a = [int(v) for v in rng.integers(0, q, tiny.n, dtype=np.uint64)]
        b = [int(v) for v in rng.integers(0, q, tiny.n, dtype=np.uint64)]
        fa, fb = tiny.ntt(pi, a), tiny.ntt(pi, b)
        prod = [(int(x) * int(y)) % q for x, y in zip(fa, fb)]
        got = [int(v) for v in tiny.ntt(pi, prod, inverse=True)]
        assert got == R.negacyclic_mul(a, b, q)


def test_galois_permutation_C10(tiny):
    """NTT-domain permutation == coefficient map X^j -> X^{jk} with X^N = -1."""
    rng = np.random.default_rng(3)
    n, q = tiny.n, tiny.primes[1]
    a = [int(v) for v in rng.integers(0, q, n, dtype=np.uint64)]
    for k in [5, 25, tiny.galois_of_rot(3), 2 * n - 1]:
        b = [0] * n
        for j in range(n):
            e = (j * k) % (2 * n)
            if e < n:
                b[e] = (b[e] + a[j]) % q
            else:
                b[e - n] = (b[e - n] - a[j]) % q
        perm = tiny.galois_perm(k)
        fa = tiny.ntt(1, a)
        assert [int(fa[perm[i]]) for i in range(n)] == [int(v) for v in tiny.ntt(1, b)]


def test_galois_of_rotation(tiny):
    n = tiny.n
    assert tiny.galois_of_rot(0) == 1
    assert tiny.galois_of_rot(1) == 5
    assert tiny.galois_of_rot(-1) == pow(5, n // 2 - 1, 2 * n)


def _read_golden_chacha():
    d = {}
    for line in open(os.path.join(GOLD, "chacha20_rfc8439.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        d[k] = v
    return d


def test_chacha20_rfc8439():
    g = _read_golden_chacha()
    key = [int(x, 16) for x in g["key"]]
    nonce = [int(x, 16) for x in g["nonce"]]
    out = O.chacha20_block(key, int(g["counter"][0]), nonce)
    assert [int(v) for v in out] == [int(x, 16) for x in g["out"]]


def test_stream_layout():
    # word idx of the stream = words 2w, 2w+1 of block idx>>3 (C5)
    seed, tag, sub = 0x1234_5678_9ABC_DEF0, 4, (7 << 32) | 3
    key = [seed & 0xFFFFFFFF, seed >> 32, tag, sub & 0xFFFFFFFF, sub >> 32, 0, 0, 0]
    for idx in [0, 5, 8, 77, 1 << 20]:
        blk = O.chacha20_block(key, idx >> 3, [0, 0, 0])
        w = idx & 7
        assert O.stream(seed, tag, sub, idx) == int(blk[2 * w]) | (int(blk[2 * w + 1]) << 32)


def test_residue_of_double():
    rng = np.random.default_rng(4)
    q = (1 << 59) - 55 * 8192 + 1
    xs = list(rng.normal(0, 1e6, 50)) + [2.5, 3.5, -2.5, 0.5, -0.5, 1e19, -3.7e21, 2.0 ** 70 + 2.0 ** 20, 1e300]
    for x in xs:
        exact = round(float(x))  # Python: exact round-half-even of the double
        assert O.residue(float(x), q) == exact % q


def test_encode_matches_50_digit_reference(tiny):
    import mpmath as mp
    mp.mp.dps = 50
    rng = np.random.default_rng(5)
    n, n0 = tiny.n, tiny.n // 2
    re, im = rng.uniform(-1, 1, n0), rng.uniform(-1, 1, n0)
    scale = 2.0 ** 40
    got = tiny.encode(re, im, scale=scale, level=0)[0]
    q0 = tiny.primes[0]
    for t in range(n):
        acc = mp.mpf(0)
        g = 1
        for j in range(n0):
            ang = -mp.pi * ((g * t) % (2 * n)) / n
            acc += mp.mpf(re[j]) * mp.cos(ang) - mp.mpf(im[j]) * mp.sin(ang)
            g = g * 5 % (2 * n)
        v = acc * mp.mpf(scale) * 2 / n
        r = int(mp.nint(v))
        assert int(got[t]) == r % q0


def test_decode_encode_roundtrip():
    P = O.Params.from_preset(W.preset("TOY12"))
    K = O.Keys(P, 11, 192, galois=[], relin=False)
    rng = np.random.default_rng(6)
    z = rng.uniform(-1, 1, P.n // 2) + 1j * rng.uniform(-1, 1, P.n // 2)
    pt = P.encode(z.real, z.imag, scale=P.scale(3), level=3)
    ct = O.encrypt(P, K, pt, 3, 1, 0, use_sk=True)
    d = O.decrypt_decode(P, K, ct)
    assert np.abs(d - z).max() < 2.0 ** -25


def test_crt_consistency_of_limbs():
    """All limbs of an encrypted-then-decrypted plaintext are residues of ONE
    small integer (RNS/CRT identity)."""
    P = O.Params.from_preset(W.preset("TINY"))
    K = O.Keys(P, 3, 8, relin=False)
    rng = np.random.default_rng(7)
    z = rng.uniform(-1, 1, P.n // 2)
    pt = P.encode(z, scale=2.0 ** 30, level=3)
    ct = O.encrypt(P, K, pt, 3, 5, 0)
    m = O.decrypt(P, K, ct)
    for t in range(P.n):
        x, Q = R.crt([int(m[i, t]) for i in range(4)], P.primes[:4])
        c = R.centred(x, Q)
        assert abs(c) < 2 ** 40
        assert all(c % P.primes[i] == int(m[i, t]) for i in range(4))
        # and it equals the plaintext coefficient up to the encryption noise
        assert abs(c - R.centred(int(pt[0, t]), P.primes[0])) < 2 ** 16
