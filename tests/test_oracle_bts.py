"""Pin of the oracle's bootstrapping (G11, C16, C17) against the
mathematics rather than itself: a bootstrapped ciphertext at level 3 must come
back at the output level and decrypt to the same message within the stated
bootstrapping precision (PAPER.md 389-390: ~22 bits for HEaaN; ours at
N = 2^12 with P16's chain: 2^-24)."""
import numpy as np

import workloads as W
from oracle import oracle as O


def test_oracle_bootstrap_precision_toy12b():
    pre = W.preset("TOY12B")
    P = O.Params.from_preset(pre)
    rots = O.bts_rotations(P, pre["bts"])
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    K = O.Keys(P, 31337, pre["h"], galois=gal)
    B = O.Bts(P, pre["bts"], W.bts_tables()[pre["bts"]["table"]])
    z = np.random.default_rng(0).uniform(-1, 1, P.n // 2)
    ct = O.encrypt(P, K, P.encode(z, scale=P.scale(3), level=3), 3, 77, 0)
    out = O.bootstrap(P, K, ct, B, 1.0)
    assert out.level == pre["bts"]["out_level"]
    err = np.abs(O.decrypt_decode(P, K, out).real - z).max()
    assert err < 2.0 ** -22, np.log2(err)
