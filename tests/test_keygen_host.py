"""Host-side KeyGen (PAPER.md 262-271 [sec 2.2.1]: KeyGen hands sk, pk and the
evaluation keys to the user; the evaluator only needs pk / evk) --
hs_ckks_keygen_host and hs_ckks_decrypt_host need no device, so their words
are checked here on the CPU against the independent oracle: the secret (C5),
pk (C6), every switching key (C7), and decryption (c0 + c1 s, C6) of an
oracle ciphertext.  The device side (hs_keys_upload) is covered by
tests/test_gpu_parity.py::test_uploaded_keys_softmax_parity."""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

hs = pytest.importorskip("paper_2410_11184_b200")


@pytest.mark.parametrize("name,rots", [("TINY", [1, -1]), ("TOY12", [1, -128, 1024]), ("P16U", [1])])
def test_host_keygen_equals_oracle(name, rots):
    pre = W.preset(name)
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    seed = 0xC0FFEE + len(name)
    HK = hs.HostKeys(P, seed, pre["h"], galois=gal)
    KO = O.Keys(PO, seed, pre["h"], galois=gal)
    assert (HK.secret() == KO.secret()).all()
    assert (HK.pk_words() == KO.pk()).all()
    for g in [0] + gal:
        assert (HK.swk(g) == KO.swk(g)).all(), g
    with pytest.raises(hs.HsError) as e:
        HK.swk(12345)
    assert e.value.code == 3   # HS_EKEY


def test_host_decrypt_equals_oracle():
    pre = W.preset("TOY12")
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    HK = hs.HostKeys(P, 77, pre["h"])
    KO = O.Keys(PO, 77, pre["h"])
    z = np.random.default_rng(1).uniform(-1, 1, P.n // 2)
    for level in (11, 4, 0):
        pt = PO.encode(z, scale=PO.scale(level), level=level)
        ct = O.encrypt(PO, KO, pt, level, 9, level)
        assert (HK.decrypt(ct.words()) == O.decrypt(PO, KO, ct)).all()
        assert np.abs(HK.decrypt_decode(ct.words()).real - z).max() < 2.0 ** -22
    # a degree-2 ciphertext (tensor) decrypts with s^2 as well: exactly
    # Dec(a (x) a) = Dec(a)^2 (negacyclic, per RNS limb; C8 tensor identity)
    a = O.encrypt(PO, KO, PO.encode(z, scale=PO.scale(3), level=3), 3, 3, 0)
    t = O.op(PO, KO, "tensor", a, a)
    m2, m1 = HK.decrypt(t.words()), HK.decrypt(a.words())
    for i in range(4):
        q = PO.primes[i]
        f1 = [int(v) for v in PO.ntt(i, m1[i])]
        f2 = [int(v) for v in PO.ntt(i, m2[i])]
        assert all(y == (x * x) % q for x, y in zip(f1, f2)), i
