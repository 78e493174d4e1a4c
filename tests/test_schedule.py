"""Schedule planner and automatic variant selection (
include/hesoftmax.h hs_softmax_schedule / hs_softmax_choose; DESIGN.md
section 10).  Host-only: the planner runs the product driver's schedule with a
level-only executor, so these run without a GPU.

Pins (none of them the planner's own arithmetic):
* the independent oracle's Softmax (oracle/, its own schedule code): output
  level, rotation count and bootstrap count of the same configuration;
* PAPER.md 444-447 [sec 5.1.4]: version B on [-128, 0] needs no main-thread
  bootstrapping; PAPER.md 608-614: Alg 1 bootstraps its main thread;
* PAPER.md 891-896 / G6: 2 log2(N0/L) rotations per aux call;
* PAPER.md 591-600 tab:SMmany: Alg 1 is the faster at 1 ciphertext, version B
  at 64, and once version B wins it keeps winning as m grows.
"""
import math

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

hs = pytest.importorskip("paper_2410_11184_b200")


@pytest.fixture(scope="module")
def tables():
    return W.poly_tables()


@pytest.fixture(scope="module")
def p16():
    pre = W.preset("P16")
    return hs.Params.from_preset(pre), pre["bts"]["out_level"]


def _cands(tables, names):
    return [dict(k=tables[t]["config"]["k"], variant=tables[t]["config"]["variant"], exp=tables[t]["exp"],
                 inv=tables[t]["inv"]) for t in names]


@pytest.mark.parametrize("m,table", [(1, "toy_n16_M2_k1_A"), (2, "toy_n16_M4_k2_A"), (2, "toy_n16_M4_k2_B"),
                                     (2, "toy_n16_M4_k2_S"), (2, "toy_n16_M4_k2_A_nt")])
def test_planner_matches_oracle_toy(tables, m, table):
    """TOY12 (no bootstrapping): the planner's output level and rotation count
    equal the oracle's run of the same Softmax."""
    pre = W.preset("TOY12" if table.endswith("k1_A") else "TOY12D")
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    tab = tables[table]
    cfg = tab["config"]
    n, k, var = 16, cfg["k"], cfg["variant"]
    K = O.Keys(PO, 5, 192, galois=O.softmax_rotation_galois(PO, n, m))
    L = (PO.n // 2) * m // n
    x = W.softmax_inputs(L, n, cfg["M"], seed=3)
    slots = O.pack(x, PO.n // 2, m)
    top = PO.n_q - 1
    sc = O.softmax_input_scale(PO, tab["exp"], top)  # G28
    cts = [O.encrypt(PO, K, PO.encode(slots[c], scale=sc, level=top), top, 9, c) for c in range(m)]
    O.ledger_reset()
    out = O.softmax(PO, K, cts, n, k, var, tab["exp"], tab["inv"])
    led = O.ledger()
    s = hs.softmax_schedule(P, n, m, k, var, tab["exp"], tab["inv"], top)
    assert s["out_level"] == out[0].level
    assert s["rotations"] == led["rot"] == k * 2 * int(math.log2(n // m))
    assert s["bts_main"] == s["bts_aux"] == 0 and s["cost"] > 0


def test_planner_matches_oracle_bootstrapped(tables):
    """Config-2 schedule (Alg 1, one ciphertext) on the N = 2^12 ring with
    P16's chain: the planner's bootstrap count and output level equal the
    oracle's (which places its bootstraps with its own code, G12)."""
    pre = W.preset("TOY12B")
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    tab = tables["p16_n256_M128_k5_A"]
    cfg = tab["config"]
    n, k, m = cfg["n"], cfg["k"], 1
    nb = n // m
    stride = (PO.n // 2) // nb
    rots = set(hs.bts_rotations(P, pre["bts"]))
    rots |= {s * (stride << i) for i in range(int(math.log2(nb))) for s in (1, -1)}
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    KO = O.Keys(PO, 17, pre["h"], galois=gal)
    BO = O.Bts(PO, pre["bts"], W.bts_tables()[pre["bts"]["table"]])
    L = (PO.n // 2) * m // n
    x = W.softmax_inputs(L, n, cfg["M"], seed=4)
    top = pre["bts"]["out_level"]
    pt = P.encode(P.pack(x, m)[0], scale=hs.softmax_input_scale(P, tab["exp"], top), level=top)
    O.ledger_reset()
    out = O.softmax_bts(PO, KO, [O.encrypt(PO, KO, pt, top, 4040, 0)], n, k, "A", tab["exp"], tab["inv"], BO)
    led = O.ledger()
    s = hs.softmax_schedule(P, n, m, k, "A", tab["exp"], tab["inv"], top, bts_out_level=top)
    assert s["bts_main"] + s["bts_aux"] == led["bts"] > 0
    assert s["bts_main"] >= 1
    assert s["out_level"] == out[0].level


def test_planner_paper_pins_p16(tables, p16):
    P, bo = p16
    tb, ta = tables["p16_n256_M128_k5_B"], tables["p16_n256_M128_k5_A"]
    # config 3: 64 ciphertexts, version B -- no main-thread bootstrap
    sb = hs.softmax_schedule(P, 256, 64, 5, "B", tb["exp"], tb["inv"], bo, bts_out_level=bo)
    assert sb["bts_main"] == 0 and sb["bts_aux"] > 0
    # 2 log2(N0/L) = 4 rotations per aux call, one shared aux ciphertext (G6)
    assert sb["rotations"] == 5 * 2 * 2
    # Alg 1 on the same batch bootstraps every main ciphertext
    sa = hs.softmax_schedule(P, 256, 64, 5, "A", ta["exp"], ta["inv"], bo, bts_out_level=bo)
    assert sa["bts_main"] > 0 and sa["bts_main"] % 64 == 0
    # config 2: one ciphertext, 8 + 8 rotations per aux call
    s2 = hs.softmax_schedule(P, 256, 1, 5, "A", ta["exp"], ta["inv"], bo, bts_out_level=bo)
    assert s2["rotations"] == 5 * 2 * 8
    # without bootstrapping the P16 chain cannot hold either (HS_ELEVEL)
    with pytest.raises(hs.HsError) as e:
        hs.softmax_schedule(P, 256, 64, 5, "B", tb["exp"], tb["inv"], bo)
    assert e.value.code == 2
    # sharding leaves the aux schedule alone: per rank the same bootstraps
    s8 = hs.softmax_schedule(P, 256, 64, 5, "B", tb["exp"], tb["inv"], bo, world=8, bts_out_level=bo)
    assert s8["bts_aux"] == sb["bts_aux"] and s8["exchanges"] == 5 and s8["out_level"] == sb["out_level"]


def test_choose_follows_tab_smmany(tables, p16):
    """tab:SMmany: Alg 1 wins at 1 ciphertext, version B at 64,
    and the choice flips once (monotone in m)."""
    P, bo = p16
    cands = _cands(tables, ["p16_n256_M128_k5_A", "p16_n256_M128_k5_B"])
    picks = []
    for m in [1, 2, 4, 8, 16, 32, 64]:
        best, sched = hs.softmax_choose(P, cands, 256, m, bo, bts_out_level=bo)
        assert sched[best]["cost"] == min(s["cost"] for s in sched)
        picks.append(cands[best]["variant"])
    assert picks[0] == "A" and picks[-1] == "B"
    flip = picks.index("B")
    assert all(p == "B" for p in picks[flip:])
    # main-thread bootstraps drive the choice: Alg 1's cost grows with m
    costs = [hs.softmax_choose(P, cands, 256, m, bo, bts_out_level=bo)[1][0]["cost"] for m in (1, 64)]
    assert costs[1] > 4 * costs[0]


def test_choose_errors(tables, p16):
    P, bo = p16
    cands = _cands(tables, ["p16_n256_M128_k5_A", "p16_n256_M128_k5_B"])
    # no bootstrapping: nothing fits the P16 chain -> HS_ELEVEL
    with pytest.raises(hs.HsError) as e:
        hs.softmax_choose(P, cands, 256, 64, bo)
    assert e.value.code == 2
    # an unfit candidate is skipped (cost = inf), the other chosen
    short = dict(cands[1], inv=cands[1]["inv"][:1], k=1)
    best, sched = hs.softmax_choose(P, [cands[0], short], 256, 1, bo, bts_out_level=bo)
    assert best in (0, 1) and all(np.isfinite(s["cost"]) or s["cost"] == float("inf") for s in sched)
    with pytest.raises(hs.HsError):
        hs.softmax_choose(P, [dict(cands[0], k=0)], 256, 1, bo, bts_out_level=bo)


def test_input_level_choice_matches_workload(tables):
    """hs_softmax_input_level (the planner's input level) for config 3 equals
    the level the workload table declares (bench.py and the reference arm's
    inventory both use it): the lowest-cost level that fits the version-B
    main thread without bootstrapping it (PAPER.md 444-447)."""
    pre = W.preset("P16")
    P = hs.Params.from_preset(pre)
    wl = W.WORKLOADS["config3"]
    tab = tables[wl["table"]]
    lv = hs.softmax_input_level(P, wl["n"], wl["m"], wl["k"], wl["variant"], tab["exp"], tab["inv"], 1,
                                pre["bts"]["out_level"])
    assert lv == wl["input_level"]
    s = hs.softmax_schedule(P, wl["n"], wl["m"], wl["k"], wl["variant"], tab["exp"], tab["inv"], lv,
                            bts_out_level=pre["bts"]["out_level"])
    assert s["bts_main"] == 0
    with pytest.raises(hs.HsError):  # one level lower no longer fits
        hs.softmax_schedule(P, wl["n"], wl["m"], wl["k"], wl["variant"], tab["exp"], tab["inv"], lv - 1,
                            bts_out_level=pre["bts"]["out_level"])


def test_reference_inventory_matches_planner(tables):
    """bench.py's reference arm weights its oracle samples by the oracle's OWN
    op inventory of the config-3 step (the exact schedule on a 2^10 ring with
    P16's chain and a bootstrap stub); its bootstrap count must equal the
    product planner's for the same workload and input level -- two independent
    implementations of G12 agreeing on the full-size schedule."""
    import bench
    wl = W.WORKLOADS["config3"]
    tab = tables[wl["table"]]
    ks, n_bts = bench.oracle_inventory(wl["input_level"])
    pre = W.preset("P16")
    P = hs.Params.from_preset(pre)
    s = hs.softmax_schedule(P, wl["n"], wl["m"], wl["k"], wl["variant"], tab["exp"], tab["inv"], wl["input_level"],
                            bts_out_level=pre["bts"]["out_level"])
    assert n_bts == s["bts_main"] + s["bts_aux"] == 7
    assert min(ks) >= 0 and max(ks) <= pre["bts"]["out_level"]
    assert sum(ks.values()) > 1000
