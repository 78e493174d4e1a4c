"""Parity of the CUDA path (through the C ABI) with the CPU oracle: every
ciphertext word must be identical, and decrypted
Softmax outputs within 2^-15 of float64 Softmax (north_star tolerance)."""
import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _hs():
    import paper_2410_11184_b200 as hs
    return hs


class Pair:
    """the same preset / keys on both sides"""

    def __init__(self, preset, seed, galois_rots=(), conj=False, relin=True):
        hs = _hs()
        self.pre = W.preset(preset)
        self.P = hs.Params.from_preset(self.pre)
        self.ctx = hs.Context(self.P, 0)
        self.PO = O.Params.from_preset(self.pre)
        gal = sorted({self.P.galois_of_rot(r) for r in galois_rots} | ({2 * self.P.n - 1} if conj else set()))
        self.gal = gal
        self.K = hs.Keys(self.ctx, seed, self.pre["h"], galois=gal, relin=relin)
        self.KO = O.Keys(self.PO, seed, self.pre["h"], galois=gal, relin=relin)
        self.top = len(self.pre["q_bits"]) - 1

    def enc(self, z, level, idx, use_sk=False, scale=None):
        hs = _hs()
        pt = self.P.encode(np.real(z), np.imag(z) if np.iscomplexobj(z) else None,
                           scale=self.P.scale(level) if scale is None else scale, level=level)
        seed = 555 + idx
        return hs.encrypt(self.K, pt, level, seed, idx, use_sk), O.encrypt(self.PO, self.KO, pt, level, seed, idx,
                                                                           use_sk)


def same(g, o):
    wg, wo = g.words(), o.words()
    assert wg.shape == wo.shape
    bad = np.argwhere(wg != wo)
    assert bad.size == 0, f"{len(bad)} words differ, first at {bad[:3].tolist()}"


@pytest.fixture(scope="module")
def toy():
    return Pair("TOY12", 4242, galois_rots=[1, -1, 3, 128, -128, 256, -256, 512, -512, 1024, -1024], conj=True)


@pytest.mark.parametrize("preset", ["TOY12", "P16U"])
def test_ntt_parity(preset):
    hs = _hs()
    pre = W.preset(preset)
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    rng = np.random.default_rng(1)
    np_ = len(P.primes)
    host = np.stack([rng.integers(0, q, P.n, dtype=np.uint64) for q in P.primes])
    dev = torch.from_numpy(host.view(np.int64)).cuda()
    ctx.ntt(dev.data_ptr(), 0, np_, inverse=False)
    got = dev.cpu().numpy().view(np.uint64)
    for i in range(np_):
        assert (got[i] == PO.ntt(i, host[i])).all(), i
    ctx.ntt(dev.data_ptr(), 0, np_, inverse=True)
    assert (dev.cpu().numpy().view(np.uint64) == host).all()


@pytest.mark.parametrize("pattern", ["max", "alternating", "impulse"])
def test_ntt_extreme_inputs_p16(pattern):
    """N = 2^16 transforms on inputs at the edges of the words' range -- every
    coefficient q - 1, alternating 0 / q - 1, a single q - 1 -- on all P16
    primes: the signed FP64 butterflies of the 42-bit primes (kernels.cu: no
    corrections inside a pass, |x| < 12 q) and the lazy integer ones must give
    the oracle's words, forward and back (C3)."""
    hs = _hs()
    pre = W.preset("P16")
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    qs = np.array(P.primes, dtype=np.uint64)
    host = np.zeros((len(qs), P.n), np.uint64)
    if pattern == "max":
        host[:] = (qs - 1)[:, None]
    elif pattern == "alternating":
        host[:, 1::2] = (qs - 1)[:, None]
    else:
        host[:, 12345] = qs - 1
    dev = torch.from_numpy(host.view(np.int64)).cuda()
    ctx.ntt(dev.data_ptr(), 0, len(qs), inverse=False)
    got = dev.cpu().numpy().view(np.uint64)
    for i in range(len(qs)):
        assert (got[i] == PO.ntt(i, host[i])).all(), i
    # the inverse of the (worst-case) spectrum -- all q - 1 -- as well
    spec = np.repeat((qs - 1)[:, None], P.n, axis=1)
    dev = torch.from_numpy(spec.copy().view(np.int64)).cuda()
    ctx.ntt(dev.data_ptr(), 0, len(qs), inverse=True)
    back = dev.cpu().numpy().view(np.uint64)
    for i in (0, 1, 13, len(qs) - 1):
        assert (PO.ntt(i, back[i]) == spec[i]).all(), i
    ctx.ntt(dev.data_ptr(), 0, len(qs), inverse=False)
    assert (dev.cpu().numpy().view(np.uint64) == spec).all()


def test_keygen_parity(toy):
    assert (toy.K.secret() == toy.KO.secret()).all()
    assert (toy.K.swk(0) == toy.KO.swk(0)).all()
    for g in toy.gal[:3]:
        assert (toy.K.swk(g) == toy.KO.swk(g)).all()


@pytest.mark.parametrize("use_sk", [False, True])
def test_encrypt_parity(toy, use_sk):
    rng = np.random.default_rng(2)
    z = rng.uniform(-1, 1, toy.P.n // 2)
    g, o = toy.enc(z, toy.top, 3, use_sk)
    same(g, o)
    hs = _hs()
    assert (hs.decrypt(toy.K, g) == O.decrypt(toy.PO, toy.KO, o)).all()
    assert np.abs(hs.decrypt_decode(toy.K, g).real - z).max() < 2.0 ** -22


def test_ops_parity(toy):
    hs = _hs()
    rng = np.random.default_rng(3)
    za, zb = rng.uniform(-1, 1, toy.P.n // 2), rng.uniform(-1, 1, toy.P.n // 2)
    a, ao = toy.enc(za, toy.top, 0)
    b, bo = toy.enc(zb, 8, 1)
    K, KO, PO = toy.K, toy.KO, toy.PO
    cases = [("add", dict(b=(b, bo))), ("sub", dict(b=(b, bo))), ("mult", dict(b=(b, bo))),
             ("tensor", dict(b=(b, bo))), ("rescale", {}), ("level_down", dict(i=5)),
             ("mult_const", dict(c=-0.731, i=9)), ("add_const", dict(c=0.3125)), ("mult_int", dict(i=-3)),
             ("rotate", dict(i=3)), ("rotate", dict(i=-128)), ("conj", {})]
    for name, kw in cases:
        bb = kw.get("b", (None, None))
        g = hs.op(K, name, a, bb[0], c=kw.get("c", 0.0), i=kw.get("i", 0))
        o = O.op(PO, KO, name, ao, bb[1], c=kw.get("c", 0.0), i=kw.get("i", 0))
        same(g, o)
    t = hs.op(K, "tensor", a, b)
    to = O.op(PO, KO, "tensor", ao, bo)
    same(hs.op(K, "relin", t), O.op(PO, KO, "relin", to))
    mask = (np.arange(toy.P.n // 2) % 5 == 0).astype(float)
    same(hs.mult_pt(a, mask, target=10), O.mult_pt(PO, ao, mask, target=10))


def test_batched_ops_parity(toy):
    """hs_ct_gather batches: each member of a batched HMult / rotation / add
    (batch x batch and batch x broadcast) equals the oracle's single op."""
    hs = _hs()
    rng = np.random.default_rng(8)
    pairs = [toy.enc(rng.uniform(-1, 1, toy.P.n // 2), 11, 20 + i) for i in range(3)]
    b, bo = toy.enc(rng.uniform(-1, 1, toy.P.n // 2), 11, 30)
    batch = hs.gather([g for g, _ in pairs])
    K, KO, PO = toy.K, toy.KO, toy.PO
    mm = hs.op(K, "mult", batch, batch)
    mb = hs.op(K, "mult", batch, b)
    rr = hs.op(K, "rotate", batch, i=-128)
    for i, (_, o) in enumerate(pairs):
        same(hs.member(mm, i), O.op(PO, KO, "mult", o, o))
        same(hs.member(mb, i), O.op(PO, KO, "mult", o, bo))
        same(hs.member(rr, i), O.op(PO, KO, "rotate", o, i=-128))


@pytest.mark.parametrize("level", [11, 7, 0])
def test_rotate_hoisted_parity(toy, level):
    """C16: every output of one hoisted ModUp is bit-exact with the oracle's."""
    hs = _hs()
    rng = np.random.default_rng(40 + level)
    z = rng.uniform(-1, 1, toy.P.n // 2)
    a, ao = toy.enc(z, level, 7)
    rots = [1, 3, -1, 128, 1024, -512, 256]
    outs = hs.rotate_hoisted(toy.K, a, rots)
    outo = O.rotate_hoisted(toy.PO, toy.KO, ao, rots)
    for g, o in zip(outs, outo):
        same(g, o)
    assert np.abs(hs.decrypt_decode(toy.K, outs[1]).real - np.roll(z, -3)).max() < 2.0 ** -20


def test_keyswitch_parity(toy):
    hs = _hs()
    rng = np.random.default_rng(4)
    P = toy.P
    for level in [toy.top, 6, 0]:
        d = np.stack([rng.integers(0, P.primes[i], P.n, dtype=np.uint64) for i in range(level + 1)])
        dd = torch.from_numpy(d.view(np.int64)).cuda()
        o0 = torch.empty_like(dd)
        o1 = torch.empty_like(dd)
        for g in [0, toy.gal[0]]:
            hs.keyswitch(toy.K, g, level, dd.data_ptr(), o0.data_ptr(), o1.data_ptr())
            torch.cuda.synchronize()
            e0, e1 = O.keyswitch(toy.PO, toy.KO, g, level, d)
            assert (o0.cpu().numpy().view(np.uint64) == e0).all()
            assert (o1.cpu().numpy().view(np.uint64) == e1).all()


@pytest.mark.parametrize("deg,a,b,gain", [(7, -2.0, 0.0, 1.0), (15, 2.0, 16.5, 0.3), (31, -1.0, 1.0, 1.0),
                                          (3, 0.25, 1.5, 1.0), (63, -1.0, 1.0, 1.7), (127, 0.5, 2.5, 1.0),
                                          (5, -3.0, 1.0, 1.0)])
def test_cheb_parity(toy, deg, a, b, gain):
    """C13 level-exact tree: words equal to the oracle's, exactly
    ceil(log2(deg+1)) levels, the input holding alpha x (G28)."""
    hs = _hs()
    rng = np.random.default_rng(deg)
    coeffs = rng.normal(0, 1, deg + 1) / (1 + np.arange(deg + 1)) ** 2
    coeffs[2] = 0.0  # exercise the zero-coefficient skip
    z = rng.uniform(a, b, toy.P.n // 2)
    g, o = toy.enc(z, toy.top, 7, scale=toy.P.scale(toy.top) * 2.0 / (b - a))
    p = dict(a=a, b=b, coeffs=coeffs)
    out = hs.cheb(toy.K, g, p, gain=gain)
    same(out, O.cheb(toy.PO, toy.KO, o, p, gain))
    assert out.level == toy.top - max(1, int(np.ceil(np.log2(deg + 1))))


def _softmax_case(tables, preset, table, m, L, tag):
    hs = _hs()
    tab = tables[table]
    cfg = tab["config"]
    n, k, M = cfg["n"], cfg["k"], cfg["M"]
    pre = W.preset(preset)
    P = hs.Params.from_preset(pre)
    PO = O.Params.from_preset(pre)
    gal = O.softmax_rotation_galois(PO, n, m)
    ctx = hs.Context(P, 0)
    seed = W.derive_seed("keys", tag)
    K, KO = hs.Keys(ctx, seed, pre["h"], galois=gal), O.Keys(PO, seed, pre["h"], galois=gal)
    x = W.softmax_inputs(L, n, M, seed=W.derive_seed("x", tag))
    slots = P.pack(x, m)
    top = len(pre["q_bits"]) - 1
    es = W.derive_seed("enc", tag)
    g_in, o_in = [], []
    sc = hs.softmax_input_scale(P, tab["exp"], top)  # G28 input contract
    assert sc == O.softmax_input_scale(PO, tab["exp"], top)
    for c in range(m):
        pt = P.encode(slots[c], scale=sc, level=top)
        g_in.append(hs.encrypt(K, pt, top, es, c))
        o_in.append(O.encrypt(PO, KO, pt, top, es, c))
    var = cfg["variant"]
    if m == 1:
        g_out = [hs.softmax_one_ctxt(K, g_in[0], n, k, var, tab["exp"], tab["inv"])]
    else:
        g_out = hs.softmax_many_ctxt(K, g_in, n, m, k, var, tab["exp"], tab["inv"])
    o_out = O.softmax(PO, KO, o_in, n, k, var, tab["exp"], tab["inv"])
    for g, o in zip(g_out, o_out):
        same(g, o)
    dec = np.stack([hs.decrypt_decode(K, c).real for c in g_out])
    y = P.unpack(dec, L, n)
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.abs(y - ref).max() < 2.0 ** -15
    return ctx.ledger()


def test_softmax_config1_parity(tables):
    led = _softmax_case(tables, "TOY12", "toy_n16_M2_k1_A", 1, 128, "config1")
    assert led["rot"] == 2 * 4


@pytest.mark.parametrize("table", ["toy_n16_M4_k2_A", "toy_n16_M4_k2_B", "toy_n16_M4_k2_S"])
def test_softmax_many_parity(tables, table):
    _softmax_case(tables, "TOY12D", table, 2, 256, "many-" + table)


def test_sharded_path_single_process(tables):
    """The world > 1 path of hs_softmax_many_ctxt on one
    GPU without ranks waiting on each other: m = 2 identical ciphertexts, so
    rank 1's partial aux sum equals rank 0's and an exchange callback that
    writes rank 0's partial into both gather slots IS the all-gather.  Rank 0's
    sharded output must equal the unsharded m = 2 run word for word."""
    hs = _hs()
    from paper_2410_11184_b200 import _lib
    tab = tables["toy_n16_M4_k2_B"]
    cfg = tab["config"]
    n, k, M = cfg["n"], cfg["k"], cfg["M"]
    pre = W.preset("TOY12D")
    P = hs.Params.from_preset(pre)
    PO = O.Params.from_preset(pre)
    gal = O.softmax_rotation_galois(PO, n, 2)
    ctx = hs.Context(P, 0)
    K = hs.Keys(ctx, 99, pre["h"], galois=gal)
    x = W.softmax_inputs((P.n // 2) * 2 // n, n, M, seed=5)
    slots = P.pack(x, 2)
    top = len(pre["q_bits"]) - 1
    pt = P.encode(slots[0], scale=hs.softmax_input_scale(P, tab["exp"], top), level=top)
    c0 = hs.encrypt(K, pt, top, 7, 0)
    c1 = hs.encrypt(K, pt, top, 7, 0)
    full = hs.softmax_many_ctxt(K, [c0, c1], n, 2, k, 1, tab["exp"], tab["inv"])
    calls = []

    def dup(user, partial, gathered, words, stream):
        calls.append(words)
        src = torch.as_tensor(_CudaBuf(partial, words), device="cuda")
        dst = torch.as_tensor(_CudaBuf(gathered, 2 * words), device="cuda")
        dst[:words].copy_(src)
        dst[words:].copy_(src)
        return 0

    fn = _lib.EXCHANGE_FN(dup)
    shard = hs.softmax_many_ctxt(K, [c0], n, 2, k, 1, tab["exp"], tab["inv"], world=2, rank=0, exchange=fn)
    assert len(calls) == k
    same(shard[0], full[0])


class _CudaBuf:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (int(ptr), False),
                                         "version": 2, "strides": None}


# ---------------------------------------------------------------- full size (N = 2^16)
@pytest.fixture(scope="module")
def p16():
    return Pair("P16U", 16161, galois_rots=[1, -128])


def test_p16_hmult_rotate_parity(p16):
    """BASELINE.json configs 2-5 ring (N = 2^16, user chain): HMult, rotation
    and rescale at the top user level, word-for-word."""
    hs = _hs()
    rng = np.random.default_rng(6)
    za, zb = rng.uniform(-1, 1, p16.P.n // 2), rng.uniform(-1, 1, p16.P.n // 2)
    a, ao = p16.enc(za, 13, 0)
    b, bo = p16.enc(zb, 13, 1)
    m = hs.op(p16.K, "mult", a, b)
    same(m, O.op(p16.PO, p16.KO, "mult", ao, bo))
    r = hs.op(p16.K, "rotate", a, i=-128)
    same(r, O.op(p16.PO, p16.KO, "rotate", ao, i=-128))
    assert np.abs(hs.decrypt_decode(p16.K, m).real - za * zb).max() < 2.0 ** -20
    # the N = 2^16 fused paths: rescale (lift + division in the NTT), constant
    # multiply / level-down (scale folded into the rescale epilogue)
    for name, kw in [("rescale", {}), ("mult_const", dict(c=-0.731, i=9)), ("level_down", dict(i=5))]:
        same(hs.op(p16.K, name, a, c=kw.get("c", 0.0), i=kw.get("i", 0)),
             O.op(p16.PO, p16.KO, name, ao, c=kw.get("c", 0.0), i=kw.get("i", 0)))


# ---------------------------------------------------------------- bootstrapping (G11)
@pytest.fixture(scope="module")
def toyb():
    hs = _hs()
    pre = W.preset("TOY12B")
    P = hs.Params.from_preset(pre)
    PO = O.Params.from_preset(pre)
    rots = set(hs.bts_rotations(P, pre["bts"]))
    for n, m in [(256, 16), (256, 1), (2048, 1)]:
        nb = n // m
        stride = (P.n // 2) // nb
        i = 0
        while (1 << i) < nb:
            rots |= {stride << i, -(stride << i)}
            i += 1
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    ctx = hs.Context(P, 0)
    K = hs.Keys(ctx, 31337, pre["h"], galois=gal)
    KO = O.Keys(PO, 31337, pre["h"], galois=gal)
    tab = W.bts_tables()[pre["bts"]["table"]]
    B = hs.Bts(ctx, pre["bts"], tab)
    BO = O.Bts(PO, pre["bts"], tab)
    return dict(P=P, PO=PO, ctx=ctx, K=K, KO=KO, B=B, BO=BO, pre=pre)


@pytest.mark.parametrize("level,bound", [(3, 1.0), (0, 1.0), (5, 300.0)])
def test_bootstrap_parity(toyb, level, bound):
    hs = _hs()
    P, PO, K, KO = toyb["P"], toyb["PO"], toyb["K"], toyb["KO"]
    rng = np.random.default_rng(level)
    z = rng.uniform(-bound, bound, P.n // 2)
    pt = P.encode(z, scale=P.scale(level), level=level)
    g = hs.encrypt(K, pt, level, 77, level)
    o = O.encrypt(PO, KO, pt, level, 77, level)
    gb = hs.bootstrap(K, toyb["B"], g, bound)
    ob = O.bootstrap(PO, KO, o, toyb["BO"], bound)
    same(gb, ob)
    assert gb.level == toyb["pre"]["bts"]["out_level"]
    err = np.abs(hs.decrypt_decode(K, gb).real - z).max() / bound
    assert err < 2.0 ** -21, np.log2(err)


@pytest.mark.parametrize("table,m", [("p16_n256_M128_k5_B", 16), ("p16_n256_M128_k5_A", 1),
                                     ("p16_n256_M128_k5_S", 1)])
def test_softmax_bts_parity(toyb, tables, table, m):
    """configs 2-3 schedule (Alg 1 / version B with bootstrapping) on the
    N = 2^12 ring with P16's chain: ciphertexts word-for-word, accuracy 2^-15."""
    hs = _hs()
    P, PO, K, KO = toyb["P"], toyb["PO"], toyb["K"], toyb["KO"]
    tab = tables[table]
    cfg = tab["config"]
    n, k = cfg["n"], cfg["k"]
    var = {"A": 0, "B": 1, "S": 2}[cfg["variant"]]
    L = (P.n // 2) * m // n
    top = toyb["pre"]["bts"]["out_level"]  # the top user level
    x = W.softmax_inputs(L, n, cfg["M"], seed=W.derive_seed("x", table))
    slots = P.pack(x, m)
    g_in, o_in = [], []
    for c in range(m):
        pt = P.encode(slots[c], scale=hs.softmax_input_scale(P, tab["exp"], top), level=top)
        g_in.append(hs.encrypt(K, pt, top, 4040, c))
        o_in.append(O.encrypt(PO, KO, pt, top, 4040, c))
    toyb["ctx"].ledger_reset()
    g_out = hs.softmax_many_ctxt(K, g_in, n, m, k, var, tab["exp"], tab["inv"], bts=toyb["B"])
    g_led = toyb["ctx"].ledger()
    O.ledger_reset()
    o_out = O.softmax_bts(PO, KO, o_in, n, k, var, tab["exp"], tab["inv"], toyb["BO"])
    # the same bootstrap schedule on both sides (G12)
    assert g_led["bts"] == O.ledger()["bts"]
    # ... and the host planner's (hs_softmax_schedule)
    plan_s = hs.softmax_schedule(P, n, m, k, var, tab["exp"], tab["inv"], top,
                                 bts_out_level=toyb["pre"]["bts"]["out_level"])
    assert plan_s["bts_main"] + plan_s["bts_aux"] == g_led["bts"]
    assert all(c.level == plan_s["out_level"] for c in g_out)
    for gc, oc in zip(g_out, o_out):
        same(gc, oc)
    dec = np.stack([hs.decrypt_decode(K, c).real for c in g_out])
    y = P.unpack(dec, L, n)
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.abs(y - ref).max() < 2.0 ** -15
    n_bts = g_led["bts"]
    assert 0 < n_bts <= (3 if var == 2 else 2) * k
    if var == 1:
        # the same Softmax as a replayable CUDA graph (hs_softmax_plan_create):
        # every replay recomputes the words above, bit for bit
        plan = hs.Plan(K, g_in, n, m, k, var, tab["exp"], tab["inv"], bts=toyb["B"])
        for _ in range(2):
            toyb["ctx"].ledger_reset()
            outs = plan.run()
            for gc, oc in zip(outs, o_out):
                same(gc, oc)
            assert toyb["ctx"].ledger()["bts"] == n_bts
        del plan


def test_softmax_newton_parity(toyb, tables):
    """Config-5 schedule (n = N0, Alg 1, degree-63 middle steps, last step =
    seed + 3 Newton steps, G24) on the N = 2^12 ring with P16's chain:
    ciphertext word-for-word against the oracle, accuracy 2^-15."""
    hs = _hs()
    P, PO, K, KO = toyb["P"], toyb["PO"], toyb["K"], toyb["KO"]
    tab = tables["toy_n2048_M32_k4_A"]
    cfg = tab["config"]
    n, k, m, L = cfg["n"], cfg["k"], 1, 1
    assert n == P.n // 2 and tab["inv"][-1]["newton"] == 3
    x = W.softmax_inputs(L, n, cfg["M"], seed=W.derive_seed("x", "toy_n2048_M32_k4_A"))
    top = toyb["pre"]["bts"]["out_level"]
    pt = P.encode(P.pack(x, m)[0], scale=hs.softmax_input_scale(P, tab["exp"], top), level=top)
    g_in = [hs.encrypt(K, pt, top, 4040, 0)]
    o_in = [O.encrypt(PO, KO, pt, top, 4040, 0)]
    toyb["ctx"].ledger_reset()
    g_out = hs.softmax_many_ctxt(K, g_in, n, m, k, 0, tab["exp"], tab["inv"], bts=toyb["B"])
    led = toyb["ctx"].ledger()
    O.ledger_reset()
    o_out = O.softmax_bts(PO, KO, o_in, n, k, 0, tab["exp"], tab["inv"], toyb["BO"])
    same(g_out[0], o_out[0])
    assert led["bts"] == O.ledger()["bts"] > 0
    y = P.unpack(hs.decrypt_decode(K, g_out[0]).real[None], L, n)
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.abs(y - ref).max() < 2.0 ** -15


def test_softmax_error_paths(tables):
    """hs_status contract of hs_softmax_many_ctxt (include/hesoftmax.h): a
    missing rotation key -> HS_EKEY, a schedule deeper than the chain without
    bootstrapping -> HS_ELEVEL, inconsistent descriptors -> HS_EINVAL, an input
    declared at the wrong scale -> HS_ESCALE, an input outside [-M, 0] with the
    debug domain check on -> HS_EDOMAIN; the context stays usable afterwards."""
    hs = _hs()
    from paper_2410_11184_b200._lib import HsError
    tab = tables["toy_n16_M2_k1_A"]
    n, k = 16, 1
    pre = W.preset("TOY12")
    P = hs.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    PO = O.Params.from_preset(pre)
    K_full = hs.Keys(ctx, 7, pre["h"], galois=O.softmax_rotation_galois(PO, n, 1))
    K_none = hs.Keys(ctx, 7, pre["h"], galois=[])
    x = W.softmax_inputs(8, n, 2.0, seed=3)
    slots = P.pack(x, 1)
    top = len(pre["q_bits"]) - 1
    sc = lambda lv: hs.softmax_input_scale(P, tab["exp"], lv)
    ct = hs.encrypt(K_full, P.encode(slots[0], scale=sc(top), level=top), top, 1, 0)
    low = hs.encrypt(K_full, P.encode(slots[0], scale=sc(4), level=4), 4, 1, 1)

    def code(fn):
        with pytest.raises(HsError) as e:
            fn()
        return e.value.code

    assert code(lambda: hs.softmax_many_ctxt(K_none, [ct], n, 1, k, 0, tab["exp"], tab["inv"])) == 3
    assert code(lambda: hs.softmax_many_ctxt(K_full, [low], n, 1, k, 0, tab["exp"], tab["inv"])) == 2
    inv_nt = [dict(p) for p in tab["inv"]]
    inv_nt[-1]["newton"] = 2
    assert code(lambda: hs.softmax_many_ctxt(K_full, [ct], n, 1, k, 1, tab["exp"], inv_nt)) == 1
    assert code(lambda: hs.softmax_many_ctxt(K_full, [ct, ct, ct], n, 3, k, 0, tab["exp"], tab["inv"])) == 1
    assert code(lambda: hs.softmax_many_ctxt(K_full, [ct, ct], n, 4, k, 0, tab["exp"], tab["inv"])) == 1
    # HS_ESCALE (C11): an input declared at the canonical scale instead of the
    # G28 input scale; a scheme op on an operand declared off-canonical
    wrong = hs.encrypt(K_full, P.encode(slots[0], scale=P.scale(top), level=top), top, 1, 2)
    wrong.set_scale(2.0 * P.scale(top))
    assert code(lambda: hs.softmax_many_ctxt(K_full, [wrong], n, 1, k, 0, tab["exp"], tab["inv"])) == 4
    ct.set_scale(sc(top))  # the right declaration passes
    assert code(lambda: hs.op(K_full, "mult", wrong, ct)) == 4  # wrong: declared at 2 Delta
    # HS_EDOMAIN (debug): an input outside [-M, 0] puts the aux sum outside the
    # first inverse-square-root interval
    ctx.debug_domain(K_full)
    bad = hs.encrypt(K_full, P.encode(P.pack(x + 2.0, 1)[0], scale=sc(top), level=top), top, 1, 3)
    assert code(lambda: hs.softmax_many_ctxt(K_full, [bad], n, 1, k, 0, tab["exp"], tab["inv"])) == 6
    ok_dbg = hs.softmax_many_ctxt(K_full, [ct], n, 1, k, 0, tab["exp"], tab["inv"])  # in-domain passes
    ctx.debug_domain(None)
    # still usable: a valid call afterwards decrypts to Softmax
    out = hs.softmax_many_ctxt(K_full, [ct], n, 1, k, 0, tab["exp"], tab["inv"])
    assert (out[0].words() == ok_dbg[0].words()).all()
    y = P.unpack(hs.decrypt_decode(K_full, out[0]).real[None], 8, n)
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.abs(y - ref).max() < 2.0 ** -15


def test_native_comm_single_rank(tables):
    """hs_comm_init (native NCCL) on one GPU: a one-rank
    communicator runs the aux-sum all-gather (a copy) on the Softmax stream,
    eagerly and captured in a CUDA-graph plan; the words equal the run
    without an exchange."""
    hs = _hs()
    tab = tables["toy_n16_M4_k2_B"]
    cfg = tab["config"]
    n, k, M, m = cfg["n"], cfg["k"], cfg["M"], 2
    pre = W.preset("TOY12D")
    P = hs.Params.from_preset(pre)
    PO = O.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    K = hs.Keys(ctx, 5, pre["h"], galois=O.softmax_rotation_galois(PO, n, m))
    x = W.softmax_inputs((P.n // 2) * m // n, n, M, seed=8)
    slots = P.pack(x, m)
    top = len(pre["q_bits"]) - 1
    sc = hs.softmax_input_scale(P, tab["exp"], top)
    cts = [hs.encrypt(K, P.encode(slots[c], scale=sc, level=top), top, 3, c) for c in range(m)]
    ref = hs.softmax_many_ctxt(K, cts, n, m, k, "B", tab["exp"], tab["inv"])
    comm = hs.Comm(ctx, 0, 1, hs.Comm.unique_id())
    got = hs.softmax_many_ctxt(K, cts, n, m, k, "B", tab["exp"], tab["inv"], comm=comm)
    for a, b in zip(got, ref):
        assert (a.words() == b.words()).all()
    plan = hs.Plan(K, cts, n, m, k, "B", tab["exp"], tab["inv"], comm=comm)
    for _ in range(2):
        for a, b in zip(plan.run(), ref):
            assert (a.words() == b.words()).all()
    del plan


def test_softmax_cube_parity(tables):
    """G27 cube-and-normalize (t = 3, PAPER.md 1645-1663) on TOY12D, n = 4,
    two ciphertexts: words equal to the oracle's, accuracy 2^-15."""
    hs = _hs()
    tab = tables["toy_n4_M4_k2_T3"]
    cfg = tab["config"]
    n, M, k, m = cfg["n"], cfg["M"], cfg["k"], 2
    pre = W.preset("TOY12D")
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    gal = O.softmax_rotation_galois(PO, n, m)
    ctx = hs.Context(P, 0)
    K, KO = hs.Keys(ctx, 21, pre["h"], galois=gal), O.Keys(PO, 21, pre["h"], galois=gal)
    L = (P.n // 2) * m // n
    x = W.softmax_inputs(L, n, M, seed=W.derive_seed("x", "cube-gpu"))
    slots = P.pack(x, m)
    top = len(pre["q_bits"]) - 1
    g_in, o_in = [], []
    for c in range(m):
        pt = P.encode(slots[c], scale=hs.softmax_input_scale(P, tab["exp"], top), level=top)
        g_in.append(hs.encrypt(K, pt, top, 13, c))
        o_in.append(O.encrypt(PO, KO, pt, top, 13, c))
    g_out = hs.softmax_many_ctxt(K, g_in, n, m, k, "T3", tab["exp"], tab["inv"])
    o_out = O.softmax(PO, KO, o_in, n, k, "T3", tab["exp"], tab["inv"])
    for g, o in zip(g_out, o_out):
        same(g, o)
    y = P.unpack(np.stack([hs.decrypt_decode(K, c).real for c in g_out]), L, n)
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.abs(y - ref).max() < 2.0 ** -15


def test_uploaded_keys_softmax_parity(tables):
    """Client / server split (PAPER.md 262-271; include/hesoftmax.h
    hs_ckks_keygen_host / hs_keys_upload): keys generated on the HOST, only
    pk + evk uploaded; the evaluating context holds no secret (decrypt and
    secret-key encryption refuse with HS_EKEY), yet the config-1 Softmax it
    computes is word for word the oracle's, and the host secret decrypts it."""
    hs = _hs()
    from paper_2410_11184_b200._lib import HsError
    tab = tables["toy_n16_M2_k1_A"]
    n, k, m, Lx = 16, 1, 1, 128
    pre = W.preset("TOY12")
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    gal = O.softmax_rotation_galois(PO, n, m)
    seed = W.derive_seed("keys", "upload")
    HK = hs.HostKeys(P, seed, pre["h"], galois=gal)
    ctx = hs.Context(P, 0)
    K = HK.upload(ctx)
    KO = O.Keys(PO, seed, pre["h"], galois=gal)
    assert (K.swk(0) == KO.swk(0)).all()
    x = W.softmax_inputs(Lx, n, 2.0, seed=W.derive_seed("x", "upload"))
    top = len(pre["q_bits"]) - 1
    pt = P.encode(P.pack(x, m)[0], scale=hs.softmax_input_scale(P, tab["exp"], top), level=top)
    g = hs.encrypt(K, pt, top, 31, 0)          # public-key encryption on the server
    o = O.encrypt(PO, KO, pt, top, 31, 0)
    same(g, o)
    for fn in (lambda: hs.decrypt(K, g), lambda: K.secret(), lambda: hs.encrypt(K, pt, top, 31, 0, use_sk=True)):
        with pytest.raises(HsError) as e:
            fn()
        assert e.value.code == 3
    out = hs.softmax_one_ctxt(K, g, n, k, "A", tab["exp"], tab["inv"])
    outo = O.softmax(PO, KO, [o], n, k, "A", tab["exp"], tab["inv"])[0]
    same(out, outo)
    y = P.unpack(HK.decrypt_decode(out).real[None], Lx, n)
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.abs(y - ref).max() < 2.0 ** -15


def test_softmax_encrypt_input_parity(tables):
    """hs_softmax_encrypt_input (G28 client step): encode at level+1
    with scale hs_softmax_input_scale(level) * q_{level+1}, public-key
    encryption, one rescale -- word for word the same steps on the oracle; the
    result decrypts to alpha_exp x with the fresh noise divided by q_{level+1}."""
    hs = _hs()
    tab = tables["p16_n256_M128_k5_B"]
    pre = W.preset("TOY12D")
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    K, KO = hs.Keys(ctx, 5150, pre["h"]), O.Keys(PO, 5150, pre["h"])
    x = W.softmax_inputs(8, 256, 128.0, seed=4)
    slots = P.pack(x, 1)[0]
    for level in (20, 9):
        g = hs.softmax_encrypt_input(K, slots, level, tab["exp"], 77, 3)
        sc = hs.softmax_input_scale(P, tab["exp"], level) * P.primes[level + 1]
        pt = PO.encode(slots, scale=sc, level=level + 1)
        o = O.op(PO, KO, "rescale", O.encrypt(PO, KO, pt, level + 1, 77, 3))
        same(g, o)
        alpha = 2.0 / (tab["exp"]["b"] - tab["exp"]["a"])
        err = np.abs(hs.decrypt_decode(K, g).real - alpha * slots).max()
        assert err < 2.0 ** -28, np.log2(err)  # vs ~2^-22 for a fresh encryption at this scale


@pytest.mark.parametrize("preset,level", [("TOY12", 9), ("P16U", 13), ("P16", 30)])
def test_digit_parallel_keyswitch_parity(preset, level):
    """SURVEY 8(f) rank 1 on one GPU: every rank's partial accumulator
    (hs_keyswitch_partial) equals the oracle's for the same digits; the
    partials of 2 and 3 ranks summed by hs_ks_acc_add and finished
    (hs_keyswitch_finish) equal the oracle's key switch; and the sharded entry
    point hs_keyswitch_sharded of rank 0 of 2 -- with an exchange callback
    standing in for the all-gather by writing rank 1's precomputed partial
    into its slot (a single-process 2-rank emulation) -- ends with the same
    words."""
    hs = _hs()
    pre = W.preset(preset)
    P, PO = hs.Params.from_preset(pre), O.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    gal = P.galois_of_rot(1)
    K = hs.Keys(ctx, 606, pre["h"], galois=[gal])
    KO = O.Keys(PO, 606, pre["h"], galois=[gal])
    rng = np.random.default_rng(level)
    d = np.stack([rng.integers(0, P.primes[i], P.n, dtype=np.uint64) for i in range(level + 1)])
    dd = torch.from_numpy(d.view(np.int64)).cuda()
    nl, ntg = level + 1, level + 1 + P.n_p
    beta = -(-nl // P.alpha)
    want0, want1 = O.keyswitch(PO, KO, gal, level, d)
    o0 = torch.empty_like(dd)
    o1 = torch.empty_like(dd)
    host = lambda t: t.cpu().numpy().view(np.uint64)
    for world in (2, 3):
        ranges = [(r * beta // world, (r + 1) * beta // world) for r in range(world)]
        parts = []
        for j0, j1 in ranges:
            acc = torch.zeros(2 * ntg * P.n, dtype=torch.int64, device="cuda")
            hs.keyswitch_partial(K, gal, level, dd.data_ptr(), j0, j1, acc.data_ptr())
            torch.cuda.synchronize()
            if preset != "P16":  # the oracle's partial (P16 at level 30: the finished words suffice)
                assert (host(acc).reshape(2, ntg, P.n) == O.ks_partial(PO, KO, gal, level, d, j0, j1)).all()
            parts.append(acc)
        tot = parts[0].clone()
        for p_ in parts[1:]:
            hs.ks_acc_add(ctx, level, tot.data_ptr(), p_.data_ptr())
        hs.keyswitch_finish(ctx, level, tot.data_ptr(), o0.data_ptr(), o1.data_ptr())
        torch.cuda.synchronize()
        assert (host(o0).reshape(nl, P.n) == want0).all() and (host(o1).reshape(nl, P.n) == want1).all(), world
    # hs_keyswitch_sharded, rank 0 of 2, single-process emulation of the all-gather
    other = torch.zeros(2 * ntg * P.n, dtype=torch.int64, device="cuda")
    hs.keyswitch_partial(K, gal, level, dd.data_ptr(), beta // 2, beta, other.data_ptr())
    torch.cuda.synchronize()
    from paper_2410_11184_b200 import _lib

    def emu(user, partial, gathered, words, stream):
        src = torch.as_tensor(_CudaBuf(partial, words), device="cuda")
        dst = torch.as_tensor(_CudaBuf(gathered, 2 * words), device="cuda")
        dst[:words].copy_(src)
        dst[words:].copy_(other)
        return 0

    fn = _lib.EXCHANGE_FN(emu)
    o0.zero_()
    o1.zero_()
    hs.keyswitch_sharded(K, gal, level, dd.data_ptr(), 0, 2, o0.data_ptr(), o1.data_ptr(), exchange=fn)
    torch.cuda.synchronize()
    assert (host(o0).reshape(nl, P.n) == want0).all() and (host(o1).reshape(nl, P.n) == want1).all()
    # the native-communicator path (uint64 sum all-reduce + mod q) on a one-rank NCCL communicator
    comm = hs.Comm(ctx, 0, 1, hs.Comm.unique_id())
    o0.zero_()
    o1.zero_()
    hs.keyswitch_sharded(K, gal, level, dd.data_ptr(), 0, 1, o0.data_ptr(), o1.data_ptr(), comm=comm)
    torch.cuda.synchronize()
    assert (host(o0).reshape(nl, P.n) == want0).all() and (host(o1).reshape(nl, P.n) == want1).all()
    del comm


@pytest.mark.parametrize("G", [2, 3])
def test_aux_split_emulation_parity(toyb, tables, G):
    """SURVEY 8(f) rank 1 inside the Softmax: with aux_split = G (world 1) every
    key switch of the shared aux thread -- relinearisation of the aux sum,
    rotate-and-sum, polynomial and lambda products, the bootstraps' EvalMod
    products and conjugations -- runs as G digit shares summed mod q (the
    sharded path's arithmetic, emulated in one process).  The config-3
    schedule (version B, m = 16, bootstrapped) on the N = 2^12 ring with
    P16's chain must give the unsplit words, ciphertext by ciphertext, and
    the same as a replayed CUDA-graph plan."""
    hs = _hs()
    P, K = toyb["P"], toyb["K"]
    tab = tables["p16_n256_M128_k5_B"]
    cfg = tab["config"]
    n, k, m = cfg["n"], cfg["k"], 16
    L = (P.n // 2) * m // n
    top = toyb["pre"]["bts"]["out_level"]
    x = W.softmax_inputs(L, n, cfg["M"], seed=W.derive_seed("x", "aux-split"))
    slots = P.pack(x, m)
    cts = [hs.softmax_encrypt_input(K, slots[c], 10, tab["exp"], 77, c) for c in range(m)]
    ref = hs.softmax_many_ctxt(K, cts, n, m, k, 1, tab["exp"], tab["inv"], bts=toyb["B"])
    toyb["ctx"].ledger_reset()
    got = hs.softmax_many_ctxt(K, cts, n, m, k, 1, tab["exp"], tab["inv"], bts=toyb["B"], aux_split=G)
    assert toyb["ctx"].ledger()["bts"] > 0
    for a, b in zip(got, ref):
        same(a, b)
    y = P.unpack(np.stack([hs.decrypt_decode(K, c).real for c in got]), L, n)
    r = np.exp(x - x.max(1, keepdims=True))
    r /= r.sum(1, keepdims=True)
    assert np.abs(y - r).max() < 2.0 ** -15


def test_allocator_hook(tables):
    """hs_context_create_ex (include/hesoftmax.h): with an
    allocator hook bound to torch's caching allocator, the library's device
    memory -- twiddle tables, keys, ciphertexts, key-switch scratch, cached
    plaintexts, bootstrap transforms, plan inputs / outputs -- comes from
    torch's pool; the words equal the default-pool context's (themselves
    oracle-pinned above) for eager Softmax, a CUDA-graph plan and a bootstrap,
    and every hook allocation is returned by the time the objects are gone."""
    import gc
    hs = _hs()
    dev = torch.cuda.current_device()
    A = hs.Allocator(lambda nb, st: torch.cuda.caching_allocator_alloc(nb, dev, st),
                     lambda p, nb, st: torch.cuda.caching_allocator_delete(p))

    def softmax_words(alloc):
        tab = tables["toy_n16_M4_k2_B"]
        n, m, k = 16, 2, tab["config"]["k"]
        pre = W.preset("TOY12D")
        P = hs.Params.from_preset(pre)
        ctx = hs.Context(P, 0, allocator=alloc)
        gal = O.softmax_rotation_galois(O.Params.from_preset(pre), n, m)
        K = hs.Keys(ctx, 99, pre["h"], galois=gal)
        x = W.softmax_inputs((P.n // 2) * m // n, n, 4.0, seed=3)
        slots = P.pack(x, m)
        top = len(pre["q_bits"]) - 1
        sc = hs.softmax_input_scale(P, tab["exp"], top)
        cts = [hs.encrypt(K, P.encode(slots[c], scale=sc, level=top), top, 5, c) for c in range(m)]
        eager = [c.words() for c in hs.softmax_many_ctxt(K, cts, n, m, k, "B", tab["exp"], tab["inv"])]
        plan = hs.Plan(K, cts, n, m, k, "B", tab["exp"], tab["inv"])
        plan.run()
        planned = [c.words() for c in plan.outputs]
        return eager, planned

    def bts_words(alloc):
        pre = W.preset("TOY12B")
        P = hs.Params.from_preset(pre)
        ctx = hs.Context(P, 0, allocator=alloc)
        gal = sorted({P.galois_of_rot(r) for r in hs.bts_rotations(P, pre["bts"])} | {2 * P.n - 1})
        K = hs.Keys(ctx, 7, pre["h"], galois=gal)
        B = hs.Bts(ctx, pre["bts"], W.bts_tables()[pre["bts"]["table"]])
        z = np.random.default_rng(0).uniform(-1, 1, P.n // 2)
        ct = hs.encrypt(K, P.encode(z, scale=P.scale(2), level=2), 2, 1, 0)
        return hs.bootstrap(K, B, ct, 1.0).words()

    base = softmax_words(None)
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_allocated(dev)
    hooked = softmax_words(A)
    assert A.n_alloc > 0
    for a, b in zip(base[0] + base[1], hooked[0] + hooked[1]):
        assert (a == b).all()
    assert (bts_words(None) == bts_words(A)).all()
    gc.collect()
    torch.cuda.synchronize()
    assert A.n_alloc == A.n_free and A.live_bytes == 0, (A.n_alloc, A.n_free, A.live_bytes)
    assert torch.cuda.memory_allocated(dev) == m0


def test_allocator_hook_failure_is_enomem(tables):
    """A hook that returns NULL makes the call fail with HS_ENOMEM (no crash,
    no fallback to the default pool); alloc without free is HS_EINVAL."""
    hs = _hs()
    P = hs.Params.from_preset(W.preset("TOY12"))
    with pytest.raises(hs.HsError) as e:
        hs.Context(P, 0, allocator=hs.Allocator(lambda nb, st: 0, lambda p, nb, st: None))
    assert e.value.code == 7
    import ctypes as C
    from paper_2410_11184_b200 import _lib as L
    half = L.Allocator(L.ALLOC_FN(lambda nb, st, u: None), L.FREE_FN(), None)
    out = C.c_void_p()
    assert L.hs_context_create_ex(P.ptr, 0, C.byref(half), C.byref(out)) == 1


@pytest.mark.timeout(900)
def test_alternative_kernel_paths_bit_exact():
    """The measured-and-selectable kernel variants give
    the same words: integer-only NTT (HS_NTT_FP=0), direct-load cols pass
    (HS_NTT_TMA=0), scalar BConv (HS_BCONV_MMA=0), and the TMA key stream of
    the hoisted inner product (HS_KS_TMA=1).  The switches are read once per
    process, so each set runs the parity tests in a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = [({"HS_NTT_FP": "0", "HS_NTT_TMA": "0", "HS_BCONV_MMA": "0"}, "ntt or p16 or keyswitch or bts_parity"),
            ({"HS_KS_TMA": "1"}, "rotate_hoisted or bootstrap_parity")]
    for env, sel in runs:
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            os.path.join(root, "tests", "test_gpu_parity.py"), "-k", sel, "-m", "gpu"],
                           cwd=root, env=dict(os.environ, **env), capture_output=True, text=True, timeout=800)
        assert r.returncode == 0, (env, r.stdout[-2000:], r.stderr[-2000:])
