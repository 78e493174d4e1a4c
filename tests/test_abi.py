"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only calls (parameters, encode, packing) agree
with the oracle's independent implementations.  No GPU needed."""
import os
import re

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "hesoftmax.h")).read()
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", src)) - {"hs_exchange_fn"})


def test_library_exports_every_declared_symbol():
    import paper_2410_11184_b200._lib as L
    syms = _header_symbols()
    assert len(syms) > 30
    for s in syms:
        assert hasattr(L._L, s), s  # ctypes lookup == dlsym


def test_library_built_for_sm100a():
    import subprocess
    so = os.path.join(ROOT, "paper_2410_11184_b200", "libhesoftmax.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", ["TINY", "TOY12", "TOY12D", "P16", "P16U"])
def test_params_parity(name):
    import paper_2410_11184_b200 as hs
    pre = W.preset(name)
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    assert P.primes == PO.primes
    for i in range(len(P.primes)):
        assert P.psi(i) == PO.psi(i)
    for l in range(P.n_q):
        assert P.scale(l) == PO.scale(l)
    for r in [0, 1, -1, 5, 1000, -(1 << 10)]:
        assert P.galois_of_rot(r) == PO.galois_of_rot(r)


def test_bad_params_rejected():
    import paper_2410_11184_b200 as hs
    with pytest.raises(hs.HsError) as e:
        hs.Params(log_n=12, q_bits=[60, 40], p_bits=[61], alpha=1, log2_anchor=[0, 0])
    assert e.value.code == 1


@pytest.mark.parametrize("name,level", [("TOY12", 11), ("TOY12", 0), ("P16U", 13)])
def test_encode_parity(name, level):
    import paper_2410_11184_b200 as hs
    pre = W.preset(name)
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    rng = np.random.default_rng(level)
    for trial in range(2):
        re_, im_ = rng.uniform(-1, 1, P.n // 2), rng.uniform(-1, 1, P.n // 2) * trial
        sc = P.scale(level) * (1 + trial * 0.37)
        assert (P.encode(re_, im_, scale=sc, level=level) == PO.encode(re_, im_, scale=sc, level=level)).all()


def test_decode_roundtrip():
    import paper_2410_11184_b200 as hs
    P = hs.Params.from_preset(W.preset("TOY12"))
    z = np.random.default_rng(0).uniform(-1, 1, P.n // 2)
    pt = P.encode(z, scale=2.0 ** 40, level=0)
    assert np.abs(P.decode(pt[0], 2.0 ** 40).real - z).max() < 2.0 ** -30  # rounding: ~sqrt(N)/2 per slot / Delta


def test_encode_overflow():
    import paper_2410_11184_b200 as hs
    P = hs.Params.from_preset(W.preset("TOY12"))
    with pytest.raises(hs.HsError) as e:
        P.encode(np.full(P.n // 2, 2.0 ** 30), scale=2.0 ** 40, level=0)
    assert e.value.code == 5


@pytest.mark.parametrize("L,n,m", [(128, 16, 1), (100, 16, 1), (256, 16, 2), (64, 256, 1), (4, 256, 64)])
def test_pack_parity(L, n, m):
    import paper_2410_11184_b200 as hs
    P = hs.Params.from_preset(W.preset("TOY12"))
    n0 = P.n // 2
    if L > n0 * m // n:
        pytest.skip("does not fit")
    x = W.softmax_inputs(L, n, 8.0, seed=L + n)
    s = P.pack(x, m)
    assert (s == O.pack(x, n0, m)).all()
    assert (P.unpack(s, L, n) == x).all()


def test_pack_rejects_indivisible():
    import paper_2410_11184_b200 as hs
    P = hs.Params.from_preset(W.preset("TOY12"))
    with pytest.raises(hs.HsError):
        P.pack(np.zeros((4, 24)), 1)   # n/m not a power of two


@pytest.mark.parametrize("name", ["TOY12B", "P16"])
def test_bts_plan_conventions_match(name):
    """rotation set and pre-scaling exponents (G11) agree with the oracle"""
    import paper_2410_11184_b200 as hs
    pre = W.preset(name)
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    cfg = pre["bts"]
    assert hs.bts_rotations(P, cfg) == O.bts_rotations(PO, cfg)
    for n_cts, n_stc in [(3, 3), (4, 3), (5, 2)]:
        c2 = dict(cfg, n_cts=n_cts, n_stc=n_stc)
        assert hs.bts_rotations(P, c2) == O.bts_rotations(PO, c2)
    for arc in [True, False]:
        for b in [0.5, 1.0, 1.5, 2.0, 64.0, 261.0, 1e6]:
            assert hs.bts_exponent(P, arc, b) == O.bts_exponent(PO, arc, b)


def test_params_reject_unsupported_key_switch_shapes():
    """hs_ckks_params (include/hesoftmax.h; round-1 advisor findings): the
    key-switch kernels take n_p == alpha special primes, hold at most 16 digit
    offsets and accumulate (dnum + 1) products in 128 bits -- descriptors
    outside those limits are refused with HS_EINVAL instead of silently
    computing wrong words."""
    import paper_2410_11184_b200 as hs
    base = W.preset("TOY12")

    def make(**kw):
        p = dict(base, **kw)
        return hs.Params.from_preset(p)

    with pytest.raises(hs.HsError) as e:
        make(p_bits=[61, 61, 61])          # n_p = 3 != alpha = 2
    assert e.value.code == 1
    with pytest.raises(hs.HsError) as e:   # 17 digits of one prime each
        make(q_bits=[60] + [40] * 16, log2_anchor=[0] * 16 + [40], alpha=1, p_bits=[61])
    assert e.value.code == 1
    make()  # the preset itself is fine
