"""ctypes wrapper of the CPU oracle (oracle/liborc.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product
package (paper_2410_11184_b200) never imports it, and the oracle shares no
code with the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liborc.so")

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")

OP = dict(add=0, sub=1, mult=2, tensor=3, relin=4, rescale=5, level_down=6, mult_const=7,
          add_const=8, mult_int=9, rotate=10, conj=11, galois=12)
LEDGER = ["hmult", "tensor", "ks", "rot", "rescale", "cmult", "pmult", "leveldown", "bts", "ntt"]


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = C.CDLL(_LIB)
        vp = C.c_void_p
        L.orc_api_params.restype = vp
        L.orc_api_params.argtypes = [C.c_int, C.c_int, i32p, C.c_int, i32p, C.c_int, i32p]
        L.orc_api_params_free.argtypes = [vp]
        L.orc_api_primes.argtypes = [vp, u64p]
        L.orc_api_psi.restype = C.c_uint64
        L.orc_api_psi.argtypes = [vp, C.c_int]
        L.orc_api_scale.restype = C.c_double
        L.orc_api_scale.argtypes = [vp, C.c_int]
        L.orc_api_ntt.argtypes = [vp, C.c_int, u64p, C.c_int]
        L.orc_api_ntt_naive.argtypes = [vp, C.c_int, u64p]
        L.orc_api_galois_perm.argtypes = [vp, C.c_int, u32p]
        L.orc_api_chacha20.argtypes = [u32p, C.c_uint32, u32p, u32p]
        L.orc_api_stream.restype = C.c_uint64
        L.orc_api_stream.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64]
        L.orc_api_residue.restype = C.c_uint64
        L.orc_api_residue.argtypes = [C.c_double, C.c_uint64]
        L.orc_api_galois_of_rot.restype = C.c_int
        L.orc_api_galois_of_rot.argtypes = [vp, C.c_int]
        L.orc_api_keygen.restype = vp
        L.orc_api_keygen.argtypes = [vp, C.c_uint64, C.c_int, i32p, C.c_int, C.c_int]
        L.orc_api_keys_free.argtypes = [vp]
        L.orc_api_secret.argtypes = [vp, vp, i64p]
        L.orc_api_pk.argtypes = [vp, vp, u64p]
        L.orc_api_swk.restype = C.c_int
        L.orc_api_swk.argtypes = [vp, vp, C.c_int, u64p]
        L.orc_api_encode.argtypes = [vp, f64p, f64p, C.c_double, C.c_int, u64p]
        L.orc_api_encode_naive.restype = C.c_double
        L.orc_api_encode_naive.argtypes = [vp, f64p, f64p, C.c_double, C.c_int]
        L.orc_api_decrypt_decode.argtypes = [vp, vp, vp, f64p, f64p]
        L.orc_api_decrypt.argtypes = [vp, vp, vp, u64p]
        L.orc_api_encrypt.restype = vp
        L.orc_api_encrypt.argtypes = [vp, vp, u64p, C.c_int, C.c_uint64, C.c_uint64, C.c_int]
        L.orc_api_ct_import.restype = vp
        L.orc_api_ct_import.argtypes = [vp, C.c_int, C.c_int, u64p]
        L.orc_api_ct_export.argtypes = [vp, vp, u64p]
        L.orc_api_ct_level.restype = C.c_int
        L.orc_api_ct_level.argtypes = [vp]
        L.orc_api_ct_ncomp.restype = C.c_int
        L.orc_api_ct_ncomp.argtypes = [vp]
        L.orc_api_ct_free.argtypes = [vp]
        L.orc_api_op.restype = vp
        L.orc_api_op.argtypes = [vp, vp, C.c_int, vp, vp, C.c_double, C.c_int]
        L.orc_api_mult_pt.restype = vp
        L.orc_api_mult_pt.argtypes = [vp, vp, f64p, f64p, C.c_int]
        L.orc_api_keyswitch.restype = C.c_int
        L.orc_api_keyswitch.argtypes = [vp, vp, C.c_int, C.c_int, u64p, u64p, u64p]
        L.orc_api_rotate_hoisted.restype = C.c_int
        L.orc_api_rotate_hoisted.argtypes = [vp, vp, vp, i32p, C.c_int, C.POINTER(vp)]
        L.orc_api_cheb.restype = vp
        L.orc_api_cheb.argtypes = [vp, vp, vp, C.c_int, C.c_double, C.c_double, f64p, C.c_double]
        L.orc_api_softmax_input_scale.restype = C.c_double
        L.orc_api_softmax_input_scale.argtypes = [vp, C.c_double, C.c_double, C.c_int]
        L.orc_api_cheb_depth.restype = C.c_int
        L.orc_api_cheb_depth.argtypes = [C.c_int]
        L.orc_api_softmax.restype = C.c_int
        L.orc_api_newton.restype = vp
        L.orc_api_newton.argtypes = [vp, vp, vp, vp]
        L.orc_api_softmax.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, i32p, f64p, f64p, f64p,
                                      C.POINTER(vp), C.POINTER(vp), C.c_int]
        L.orc_api_ledger.argtypes = [C.POINTER(C.c_long)]
        _lib = L
    return _lib


class Params:
    """An oracle parameter set (C1, C2, C12)."""

    def __init__(self, log_n, q_bits, p_bits, alpha, log2_anchor):
        L = lib()
        self.log_n, self.n = log_n, 1 << log_n
        self.q_bits, self.p_bits = list(q_bits), list(p_bits)
        self.n_q, self.n_p, self.alpha = len(q_bits), len(p_bits), alpha
        self.ptr = L.orc_api_params(log_n, self.n_q, np.array(q_bits, np.int32), self.n_p,
                                    np.array(p_bits, np.int32), alpha, np.array(log2_anchor, np.int32))
        assert self.ptr
        pr = np.zeros(self.n_q + self.n_p, np.uint64)
        L.orc_api_primes(self.ptr, pr)
        self.primes = [int(x) for x in pr]
        self.dnum = (self.n_q + alpha - 1) // alpha

    @classmethod
    def from_preset(cls, pre: dict):
        return cls(pre["log_n"], pre["q_bits"], pre["p_bits"], pre["alpha"], pre["log2_anchor"])

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.orc_api_params_free(self.ptr)
            self.ptr = None

    def psi(self, i):
        return int(lib().orc_api_psi(self.ptr, i))

    def scale(self, level):
        return float(lib().orc_api_scale(self.ptr, level))

    def ntt(self, pi, a, inverse=False):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().orc_api_ntt(self.ptr, pi, a, 1 if inverse else 0)
        return a

    def ntt_naive(self, pi, a):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().orc_api_ntt_naive(self.ptr, pi, a)
        return a

    def galois_perm(self, k):
        p = np.zeros(self.n, np.uint32)
        lib().orc_api_galois_perm(self.ptr, k, p)
        return p

    def galois_of_rot(self, r):
        return int(lib().orc_api_galois_of_rot(self.ptr, r))

    def encode(self, re, im=None, scale=None, level=0):
        re = np.ascontiguousarray(re, np.float64)
        im = np.zeros_like(re) if im is None else np.ascontiguousarray(im, np.float64)
        out = np.zeros((level + 1) * self.n, np.uint64)
        lib().orc_api_encode(self.ptr, re, im, scale, level, out)
        return out.reshape(level + 1, self.n)


class Keys:
    def __init__(self, params: Params, seed: int, h: int, galois=(), relin=True):
        self.P = params
        g = np.array(list(galois), np.int32) if len(galois) else np.zeros(1, np.int32)
        self.galois = list(galois)
        self.ptr = lib().orc_api_keygen(params.ptr, seed, h, g, len(galois), 1 if relin else 0)

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.orc_api_keys_free(self.ptr)
            self.ptr = None

    def secret(self):
        s = np.zeros(self.P.n, np.int64)
        lib().orc_api_secret(self.P.ptr, self.ptr, s)
        return s

    def pk(self):
        o = np.zeros(2 * self.P.n_q * self.P.n, np.uint64)
        lib().orc_api_pk(self.P.ptr, self.ptr, o)
        return o.reshape(2, self.P.n_q, self.P.n)

    def swk(self, galois):
        P = self.P
        o = np.zeros(P.dnum * 2 * (P.n_q + P.n_p) * P.n, np.uint64)
        assert lib().orc_api_swk(P.ptr, self.ptr, galois, o) == 0
        return o.reshape(P.dnum, 2, P.n_q + P.n_p, P.n)


class Ct:
    def __init__(self, params: Params, ptr):
        assert ptr, "oracle op failed"
        self.P, self.ptr = params, ptr

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.orc_api_ct_free(self.ptr)
            self.ptr = None

    @property
    def level(self):
        return lib().orc_api_ct_level(self.ptr)

    @property
    def ncomp(self):
        return lib().orc_api_ct_ncomp(self.ptr)

    def words(self):
        w = np.zeros(self.ncomp * (self.level + 1) * self.P.n, np.uint64)
        lib().orc_api_ct_export(self.P.ptr, self.ptr, w)
        return w.reshape(self.ncomp, self.level + 1, self.P.n)

    @classmethod
    def from_words(cls, params, words):
        words = np.ascontiguousarray(words, np.uint64)
        nc, l1, _ = words.shape
        return cls(params, lib().orc_api_ct_import(params.ptr, l1 - 1, nc, words.ravel()))


def encrypt(P: Params, K: Keys, pt, level, seed, idx, use_sk=False) -> Ct:
    pt = np.ascontiguousarray(pt, np.uint64).reshape(-1)
    return Ct(P, lib().orc_api_encrypt(P.ptr, K.ptr, pt, level, seed, idx, 1 if use_sk else 0))


def decrypt_decode(P: Params, K: Keys, ct: Ct):
    re = np.zeros(P.n // 2)
    im = np.zeros(P.n // 2)
    lib().orc_api_decrypt_decode(P.ptr, K.ptr, ct.ptr, re, im)
    return re + 1j * im


def decrypt(P: Params, K: Keys, ct: Ct):
    o = np.zeros((ct.level + 1) * P.n, np.uint64)
    lib().orc_api_decrypt(P.ptr, K.ptr, ct.ptr, o)
    return o.reshape(ct.level + 1, P.n)


def op(P: Params, K, name, a: Ct, b: Ct = None, c: float = 0.0, i: int = 0) -> Ct:
    return Ct(P, lib().orc_api_op(P.ptr, K.ptr if K is not None else None, OP[name], a.ptr,
                                  b.ptr if b is not None else None, c, i))


def mult_pt(P: Params, a: Ct, re, im=None, target=None) -> Ct:
    re = np.ascontiguousarray(re, np.float64)
    im = np.zeros_like(re) if im is None else np.ascontiguousarray(im, np.float64)
    return Ct(P, lib().orc_api_mult_pt(P.ptr, a.ptr, re, im, a.level - 1 if target is None else target))


def keyswitch(P: Params, K: Keys, galois, level, d):
    d = np.ascontiguousarray(d, np.uint64).reshape(-1)
    o0 = np.zeros((level + 1) * P.n, np.uint64)
    o1 = np.zeros_like(o0)
    assert lib().orc_api_keyswitch(P.ptr, K.ptr, galois, level, d, o0, o1) == 0
    return o0.reshape(level + 1, P.n), o1.reshape(level + 1, P.n)


def ks_partial(P: Params, K: Keys, galois, level, d, j0, j1):
    """Digit-parallel key switch: the C7 accumulator
    [2][level+1+n_p][N] of the digits [j0, j1) only."""
    L = lib()
    L.orc_api_ks_partial.restype = C.c_int
    L.orc_api_ks_partial.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, u64p, C.c_int, C.c_int, u64p]
    d = np.ascontiguousarray(d, np.uint64).reshape(-1)
    ntg = level + 1 + P.n_p
    acc = np.zeros(2 * ntg * P.n, np.uint64)
    assert L.orc_api_ks_partial(P.ptr, K.ptr, galois, level, d, j0, j1, acc) == 0
    return acc.reshape(2, ntg, P.n)


def ks_finish(P: Params, level, acc):
    """ModDown of a (summed) key-switch accumulator -> (out0, out1)."""
    L = lib()
    L.orc_api_ks_finish.argtypes = [C.c_void_p, C.c_int, u64p, u64p, u64p]
    acc = np.ascontiguousarray(acc, np.uint64).reshape(-1)
    o0 = np.zeros((level + 1) * P.n, np.uint64)
    o1 = np.zeros_like(o0)
    L.orc_api_ks_finish(P.ptr, level, acc, o0, o1)
    return o0.reshape(level + 1, P.n), o1.reshape(level + 1, P.n)


def ext_primes(P: Params, level):
    """primes of the extended basis Q_level u P (the accumulator's limbs)"""
    return P.primes[: level + 1] + P.primes[P.n_q:]


def rotate_hoisted(P: Params, K: Keys, a: Ct, rots):
    """C16: every rotation in rots from ONE ModUp of a's c1."""
    r = np.ascontiguousarray(rots, np.int32)
    out = (C.c_void_p * len(rots))()
    assert lib().orc_api_rotate_hoisted(P.ptr, K.ptr, a.ptr, r, len(rots), out) == 0, "missing rotation key"
    return [Ct(P, out[i]) for i in range(len(rots))]


def newton_step(P: Params, K: Keys, xh: Ct, y: Ct) -> Ct:
    """One Newton inverse-square-root step y (3 - x y^2)/2 from xh = x/2
    (PAPER.md 1313-1316; G24)."""
    return Ct(P, lib().orc_api_newton(P.ptr, K.ptr, xh.ptr, y.ptr))


def cheb(P: Params, K: Keys, x: Ct, poly: dict, gain: float = 1.0) -> Ct:
    """C13: x holds alpha x (alpha = 2/(b-a), G28); returns gain * p(x)."""
    c = np.ascontiguousarray(poly["coeffs"], np.float64)
    return Ct(P, lib().orc_api_cheb(P.ptr, K.ptr, x.ptr, len(c) - 1, poly["a"], poly["b"], c, float(gain)))


def softmax_input_scale(P: Params, exp_poly: dict, level: int) -> float:
    """G28: the Softmax reads its input x encoded at Delta_level * 2/(b-a) of the
    exp table (the exp polynomial's affine factor folded into the encoding)."""
    return float(lib().orc_api_softmax_input_scale(P.ptr, exp_poly["a"], exp_poly["b"], level))


def cheb_depth(deg):
    return lib().orc_api_cheb_depth(deg)


# S: square-and-normalize (G26); T3: cube-and-normalize (G27)
VARIANT = {"A": 0, "B": 1, "S": 2, "T3": 3, 0: 0, 1: 1, 2: 2, 3: 3}


def softmax(P: Params, K: Keys, cts, n, k, variant, exp_poly, inv_polys):
    variant = VARIANT[variant]
    polys = [exp_poly] + list(inv_polys)
    assert len(inv_polys) == k
    degs = np.array([len(p["coeffs"]) - 1 for p in polys], np.int32)
    a_s = np.array([p["a"] for p in polys], np.float64)
    b_s = np.array([p["b"] for p in polys], np.float64)
    co = np.concatenate([np.asarray(p["coeffs"], np.float64) for p in polys])
    m = len(cts)
    ins = (C.c_void_p * m)(*[c.ptr for c in cts])
    outs = (C.c_void_p * m)()
    rc = lib().orc_api_softmax(P.ptr, K.ptr, n, m, k, variant, degs, a_s, b_s, co, ins, outs,
                               int(inv_polys[-1].get("newton", 0)))
    if rc != 0:
        raise RuntimeError(f"oracle softmax failed rc={rc}")
    return [Ct(P, outs[i]) for i in range(m)]


def set_threads(n: int):
    """OpenMP threads the oracle uses (1 = the paper's single-thread setting)."""
    lib().orc_api_set_threads(int(n))


def max_threads() -> int:
    return int(lib().orc_api_max_threads())


def ledger():
    a = (C.c_long * len(LEDGER))()
    lib().orc_api_ledger(a)
    return dict(zip(LEDGER, list(a)))


def ledger_reset():
    lib().orc_api_ledger_reset()


def chacha20_block(key, counter, nonce):
    out = np.zeros(16, np.uint32)
    lib().orc_api_chacha20(np.array(key, np.uint32), counter, np.array(nonce, np.uint32), out)
    return out


def stream(seed, tag, sub, idx):
    return int(lib().orc_api_stream(seed, tag, sub, idx))


def residue(x, q):
    return int(lib().orc_api_residue(x, q))


# ---------------------------------------------------------------- packing (a13)
def pack(x, n0, m):
    """PAPER.md 94-131: x[L, n] -> m slot vectors of N0.

    nb = n/m coordinate blocks per ciphertext, stride = N0/nb; instance o's
    coordinate i goes to ciphertext i // nb, slot (i % nb) * stride + o.
    Unused lanes (o >= L) carry the input x = 0 (G9)."""
    L, n = x.shape
    nb = n // m
    stride = n0 // nb
    assert n % m == 0 and L <= stride
    out = np.zeros((m, n0))
    for i in range(n):
        out[i // nb, (i % nb) * stride: (i % nb) * stride + L] = x[:, i]
    return out


def unpack(slots, L, n):
    m, n0 = slots.shape
    nb = n // m
    stride = n0 // nb
    y = np.zeros((L, n))
    for i in range(n):
        y[:, i] = slots[i // nb, (i % nb) * stride: (i % nb) * stride + L]
    return y


def softmax_rotation_galois(P, n, m):
    """Galois elements the aux thread needs: rotations by -+stride*2^i (Alg 2)."""
    nb = n // m
    stride = (P.n // 2) // nb
    out = set()
    i = 0
    while (1 << i) < nb:
        out.add(P.galois_of_rot(stride << i))
        out.add(P.galois_of_rot(-(stride << i)))
        i += 1
    return sorted(out)


# ---------------------------------------------------------------- bootstrapping (G11)
def _bts_sigs():
    L = lib()
    if getattr(L, "_bts_ready", False):
        return L
    vp = C.c_void_p
    L.orc_api_bts_new.restype = vp
    L.orc_api_bts_new.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, f64p, C.c_int]
    L.orc_api_bts_free.argtypes = [vp]
    L.orc_api_bts_rotations.restype = C.c_int
    L.orc_api_bts_rotations.argtypes = [vp, C.c_int, C.c_int, i32p, C.c_int]
    L.orc_api_bootstrap.restype = vp
    L.orc_api_bootstrap.argtypes = [vp, vp, vp, vp, C.c_double]
    L.orc_api_bts_exponent.restype = C.c_int
    L.orc_api_bts_exponent.argtypes = [vp, C.c_int, C.c_double]
    L.orc_api_softmax_bts.restype = C.c_int
    L.orc_api_softmax_bts.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, i32p, f64p, f64p, f64p,
                                      C.POINTER(vp), C.POINTER(vp), vp, C.c_int]
    L._bts_ready = True
    return L


def bts_rotations(P: Params, cfg: dict):
    """cfg: a preset's "bts" entry (n_cts, n_stc)"""
    out = np.zeros(512, np.int32)
    n = _bts_sigs().orc_api_bts_rotations(P.ptr, cfg["n_cts"], cfg["n_stc"], out, 512)
    return [int(v) for v in out[:n]]


class Bts:
    """Precomputed bootstrapping plans (diagonals encoded in quad precision).

    cfg: a preset's "bts" entry {n_cts, n_stc, arcsine, out_level}; table: the
    EvalMod cosine table {K, r, coeffs}."""

    def __init__(self, P: Params, cfg: dict, table: dict):
        c = np.ascontiguousarray(table["coeffs"], np.float64)
        self.P, self.cfg = P, cfg
        self.ptr = _bts_sigs().orc_api_bts_new(P.ptr, table["K"], table["r"], cfg["n_cts"], cfg["n_stc"],
                                               1 if cfg["arcsine"] else 0, len(c) - 1, c, cfg["out_level"])
        assert self.ptr, "bootstrapping chain does not match the parameter set"

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.orc_api_bts_free(self.ptr)
            self.ptr = None


def bootstrap(P: Params, K: Keys, ct: Ct, bts: Bts, bound: float = 1.0) -> Ct:
    """bound: upper bound on |slot values| (selects the pre-scaling exponent, G11)"""
    return Ct(P, _bts_sigs().orc_api_bootstrap(P.ptr, K.ptr, ct.ptr, bts.ptr, bound))


def bts_exponent(P: Params, arcsine: bool, bound: float) -> int:
    return int(_bts_sigs().orc_api_bts_exponent(P.ptr, 1 if arcsine else 0, bound))


def softmax_bts(P: Params, K: Keys, cts, n, k, variant, exp_poly, inv_polys, bts: Bts):
    variant = VARIANT[variant]
    polys = [exp_poly] + list(inv_polys)
    degs = np.array([len(p["coeffs"]) - 1 for p in polys], np.int32)
    a_s = np.array([p["a"] for p in polys], np.float64)
    b_s = np.array([p["b"] for p in polys], np.float64)
    co = np.concatenate([np.asarray(p["coeffs"], np.float64) for p in polys])
    m = len(cts)
    ins = (C.c_void_p * m)(*[c.ptr for c in cts])
    outs = (C.c_void_p * m)()
    rc = _bts_sigs().orc_api_softmax_bts(P.ptr, K.ptr, n, m, k, variant, degs, a_s, b_s, co, ins, outs,
                                         bts.ptr if bts is not None else None,
                                         int(inv_polys[-1].get("newton", 0)))
    if rc != 0:
        raise RuntimeError(f"oracle softmax failed rc={rc}")
    return [Ct(P, outs[i]) for i in range(m)]


# ---------------------------------------------------------------- level trace (test hook)
TRACE_EVENTS = ["exp", "square", "poly", "mask", "main", "bts_main", "bts_aux", "lambda"]


def trace(on: bool):
    """Record (event, j, level_in, level_out) for every step of the next Softmax."""
    lib().orc_api_trace(1 if on else 0)


def trace_get():
    L = lib()
    L.orc_api_trace_get.restype = C.c_int
    buf = np.zeros(512 * 4, np.int32)
    n = L.orc_api_trace_get(buf.ctypes.data_as(C.POINTER(C.c_int)), 512)
    return [(TRACE_EVENTS[e], int(j), int(a), int(b)) for e, j, a, b in buf[: 4 * n].reshape(n, 4)]


# ---------------------------------------------------------------- op inventory (bench.py --impl reference)
def ks_levels():
    a = (C.c_long * 64)()
    lib().orc_api_ks_levels(a)
    return list(a)


def softmax_inventory(P: Params, K: Keys, cts, n, k, variant, exp_poly, inv_polys, out_level):
    """The Softmax schedule with a zero-returning bootstrap stub: fills the
    ledger / per-level key-switch counters of one step (not for parity)."""
    variant = VARIANT[variant]
    polys = [exp_poly] + list(inv_polys)
    degs = np.array([len(p["coeffs"]) - 1 for p in polys], np.int32)
    a_s = np.array([p["a"] for p in polys], np.float64)
    b_s = np.array([p["b"] for p in polys], np.float64)
    co = np.concatenate([np.asarray(p["coeffs"], np.float64) for p in polys])
    m = len(cts)
    ins = (C.c_void_p * m)(*[c.ptr for c in cts])
    outs = (C.c_void_p * m)()
    L = lib()
    L.orc_api_softmax_inventory.restype = C.c_int
    L.orc_api_softmax_inventory.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, i32p, f64p,
                                            f64p, f64p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int,
                                            C.c_int]
    rc = L.orc_api_softmax_inventory(P.ptr, K.ptr, n, m, k, variant, degs, a_s, b_s, co, ins, outs, out_level,
                                     int(inv_polys[-1].get("newton", 0)))
    if rc != 0:
        raise RuntimeError(f"oracle softmax inventory failed rc={rc}")
    return [Ct(P, outs[i]) for i in range(m)]
