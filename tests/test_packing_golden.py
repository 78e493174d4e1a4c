"""Packing pinned to the layouts PAPER.md displays
(tests/golden/packing.txt: sec 4.1 one-ciphertext vector, PAPER.md 101-104;
sec 4.2 ctxt_j, PAPER.md 121-129; the SPEC's instantiated examples), for both
the oracle's pack and the library's hs_pack.  Coordinate i of instance l
carries the unique value 100 i + l, so a transposed or shifted layout fails."""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "packing.txt")


def cases():
    out, cur = [], None
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f = line.split()
        if f[0] in ("one", "many"):
            kv = dict(t.split("=") for t in f[1:])
            cur = dict(kind=f[0], **{k: int(v) for k, v in kv.items()}, rows=[])
            out.append(cur)
        else:
            cur["rows"].append([0.0 if t == "0" else 100 * int(t.split(".")[0]) + int(t.split(".")[1])
                                for t in f[1:]])
    return out


@pytest.mark.parametrize("case", cases(), ids=lambda c: f"{c['kind']}-N0{c['N0']}-n{c['n']}-L{c['L']}-m{c['m']}")
def test_pack_matches_paper_layout(case):
    n0, n, L, m = case["N0"], case["n"], case["L"], case["m"]
    # x[l-1, i-1] = 100 i + l
    x = np.array([[100.0 * i + l for i in range(1, n + 1)] for l in range(1, L + 1)])
    want = np.array(case["rows"])
    assert want.shape == (m, n0)
    got_o = O.pack(x, n0, m)
    assert (got_o == want).all(), got_o
    assert (O.unpack(got_o, L, n) == x).all()
    import paper_2410_11184_b200 as hs
    from paper_2410_11184_b200 import _lib as L_
    out = np.zeros(m * n0)
    hs.check(L_.hs_pack(np.ascontiguousarray(x).ravel(), L, n, m, n0, out))
    assert (out.reshape(m, n0) == want).all(), out
    back = np.zeros(L * n)
    hs.check(L_.hs_unpack(out, L, n, m, n0, back))
    assert (back.reshape(L, n) == x).all()
