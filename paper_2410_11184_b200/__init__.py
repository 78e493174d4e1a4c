"""B200-native RNS-CKKS Softmax (arXiv 2410.11184) -- Python binding.

Same names as the C ABI in include/hesoftmax.h; this layer only marshals
arguments.  PyTorch supplies streams (``torch.cuda.current_stream()``) and,
for the sharded many-ciphertext case, the process group that performs the
all-gather of partial aux sums.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from ._lib import HsError, check

__all__ = ["Params", "Context", "Allocator", "torch_allocator", "Keys", "Ciphertext", "HsError", "softmax_one_ctxt", "softmax_many_ctxt"]


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return None
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def _ints(v):
    a = (C.c_int * len(v))(*v)
    return a


class Params:
    """hs_ckks_params: primes (C1), psi (C2), canonical scales (C12)."""

    def __init__(self, log_n, q_bits, p_bits, alpha, log2_anchor, **_):
        self._keep = [_ints(q_bits), _ints(p_bits), _ints(log2_anchor)]
        d = L.ParamsDesc(log_n, len(q_bits), self._keep[0], len(p_bits), self._keep[1], alpha, self._keep[2])
        out = C.c_void_p()
        check(L.hs_ckks_params(C.byref(d), C.byref(out)))
        self.ptr = out
        self.log_n, self.n = log_n, 1 << log_n
        self.n_q, self.n_p, self.alpha = len(q_bits), len(p_bits), alpha
        self.dnum = (self.n_q + alpha - 1) // alpha
        pr = np.zeros(self.n_q + self.n_p, np.uint64)
        check(L.hs_params_primes(self.ptr, pr))
        self.primes = [int(x) for x in pr]

    @classmethod
    def from_preset(cls, pre):
        return cls(**pre)

    def __del__(self):
        if getattr(self, "ptr", None):
            L.hs_params_destroy(self.ptr)
            self.ptr = None

    def psi(self, i):
        return int(L.hs_params_psi(self.ptr, i))

    def scale(self, level):
        return float(L.hs_params_scale(self.ptr, level))

    def galois_of_rot(self, r):
        return int(L.hs_galois_of_rot(self.ptr, r))

    def encode(self, re, im=None, scale=None, level=0):
        re = np.ascontiguousarray(re, np.float64)
        imp = None if im is None else np.ascontiguousarray(im, np.float64)
        out = np.zeros((level + 1) * self.n, np.uint64)
        check(L.hs_ckks_encode(self.ptr, re, None if imp is None else imp.ctypes.data_as(C.c_void_p),
                               len(re), level, scale, out))
        return out.reshape(level + 1, self.n)

    def decode(self, q0_coeffs, scale):
        re, im = np.zeros(self.n // 2), np.zeros(self.n // 2)
        check(L.hs_ckks_decode(self.ptr, np.ascontiguousarray(q0_coeffs, np.uint64), scale, re, im, self.n // 2))
        return re + 1j * im

    def pack(self, x, m):
        x = np.ascontiguousarray(x, np.float64)
        Lx, n = x.shape
        out = np.zeros(m * self.n // 2)
        check(L.hs_pack(x.ravel(), Lx, n, m, self.n // 2, out))
        return out.reshape(m, self.n // 2)

    def unpack(self, slots, Lx, n):
        slots = np.ascontiguousarray(slots, np.float64)
        m = slots.shape[0]
        out = np.zeros(Lx * n)
        check(L.hs_unpack(slots.ravel(), Lx, n, m, self.n // 2, out))
        return out.reshape(Lx, n)


class Allocator:
    """hs_allocator (include/hesoftmax.h) from two Python callables:
    alloc(nbytes, stream) -> device pointer (int; 0 = failure) and
    free(ptr, nbytes, stream).  Keeps live-allocation counters.  The ctypes
    callbacks live as long as this object; a Context holds a reference."""

    def __init__(self, alloc, free):
        self.n_alloc = self.n_free = self.live_bytes = 0

        def _a(nbytes, stream, user):
            try:
                p = int(alloc(int(nbytes), int(stream or 0)))
            except Exception:
                return None
            if p:
                self.n_alloc += 1
                self.live_bytes += int(nbytes)
            return p or None

        def _f(ptr, nbytes, stream, user):
            try:
                free(int(ptr), int(nbytes), int(stream or 0))
                self.n_free += 1
                self.live_bytes -= int(nbytes)
            except Exception:
                pass

        self._cb = (L.ALLOC_FN(_a), L.FREE_FN(_f))
        self.struct = L.Allocator(self._cb[0], self._cb[1], None)


_TORCH_ALLOCATOR = None


def torch_allocator():
    """The library's device memory served by torch's caching allocator
    (SURVEY.md 8(b)): one process-wide Allocator, never freed."""
    global _TORCH_ALLOCATOR
    if _TORCH_ALLOCATOR is None:
        import torch

        def alloc(nbytes, stream):
            return torch.cuda.caching_allocator_alloc(nbytes, torch.cuda.current_device(), stream)

        def free(ptr, nbytes, stream):
            torch.cuda.caching_allocator_delete(ptr)

        _TORCH_ALLOCATOR = Allocator(alloc, free)
    return _TORCH_ALLOCATOR


class Context:
    def __init__(self, params: Params, device: int = 0, allocator=None):
        """allocator: None (the device's stream-ordered pool), "torch"
        (torch_allocator()) or an Allocator -- hs_context_create_ex."""
        self.params = params
        if isinstance(allocator, str):
            if allocator != "torch":
                raise ValueError(f"unknown allocator {allocator!r}")
            allocator = torch_allocator()
        self.allocator = allocator
        out = C.c_void_p()
        if allocator is None:
            check(L.hs_context_create(params.ptr, device, C.byref(out)))
        else:
            check(L.hs_context_create_ex(params.ptr, device, C.byref(allocator.struct), C.byref(out)))
        self.ptr = out

    def __del__(self):
        if getattr(self, "ptr", None):
            L.hs_context_destroy(self.ptr)
            self.ptr = None

    def ledger(self):
        a = (C.c_int64 * len(L.LEDGER))()
        check(L.hs_ledger_get(self.ptr, a, len(L.LEDGER)))
        return dict(zip(L.LEDGER, list(a)))

    def ledger_reset(self):
        check(L.hs_ledger_reset(self.ptr))

    def debug_domain(self, keys=None):
        """hs_ctx_debug_domain: eager Softmax calls check the aux sums against
        the polynomial intervals (HS_EDOMAIN); keys must hold the secret."""
        check(L.hs_ctx_debug_domain(self.ptr, keys.ptr if keys is not None else None))

    def ntt(self, data_ptr, prime_index, n_limbs, inverse=False, stream=None):
        check(L.hs_ntt(self.ptr, prime_index, n_limbs, C.c_void_p(data_ptr), 1 if inverse else 0, _stream(stream)))


class Keys:
    def __init__(self, ctx: Context, seed: int, h: int, galois=(), relin=True, stream=None):
        self.ctx = ctx
        g = np.array(list(galois) or [0], np.int32)
        out = C.c_void_p()
        check(L.hs_ckks_keygen(ctx.ptr, seed, h, g, len(galois), 1 if relin else 0, _stream(stream), C.byref(out)))
        self.ptr = out

    def __del__(self):
        if getattr(self, "ptr", None):
            L.hs_keys_destroy(self.ptr)
            self.ptr = None

    def swk(self, galois):
        P = self.ctx.params
        o = np.zeros(P.dnum * 2 * (P.n_q + P.n_p) * P.n, np.uint64)
        check(L.hs_keys_export_swk(self.ctx.ptr, self.ptr, galois, o))
        return o.reshape(P.dnum, 2, P.n_q + P.n_p, P.n)

    def secret(self):
        s = np.zeros(self.ctx.params.n, np.int64)
        check(L.hs_keys_export_secret(self.ctx.ptr, self.ptr, s))
        return s


class HostKeys:
    """hs_ckks_keygen_host: the client's KeyGen on the host (PAPER.md 262-271):
    secret, public key and evaluation keys as host objects.  upload(ctx) gives
    the server a device key set WITHOUT the secret (hs_keys_upload);
    decrypt_decode(ct) decrypts exported words with the host secret."""

    def __init__(self, params: Params, seed: int, h: int, galois=(), relin=True):
        self.params = params
        g = np.array(list(galois) or [0], np.int32)
        sk, pk, evk = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(L.hs_ckks_keygen_host(params.ptr, seed, h, g, len(galois), 1 if relin else 0, C.byref(sk),
                                    C.byref(pk), C.byref(evk)))
        self.sk, self.pk, self.evk = sk, pk, evk

    def __del__(self):
        for name, fn in (("sk", "hs_secret_key_destroy"), ("pk", "hs_public_key_destroy"),
                         ("evk", "hs_eval_keys_destroy")):
            if getattr(self, name, None):
                getattr(L, fn)(getattr(self, name))
                setattr(self, name, None)

    def upload(self, ctx: Context, with_pk=True, stream=None) -> "Keys":
        out = C.c_void_p()
        check(L.hs_keys_upload(ctx.ptr, self.pk if with_pk else None, self.evk, _stream(stream), C.byref(out)))
        k = Keys.__new__(Keys)
        k.ctx, k.ptr = ctx, out
        return k

    def secret(self):
        s = np.zeros(self.params.n, np.int64)
        check(L.hs_secret_key_export(self.sk, s))
        return s

    def swk(self, galois):
        P = self.params
        o = np.zeros(P.dnum * 2 * (P.n_q + P.n_p) * P.n, np.uint64)
        check(L.hs_eval_keys_export(self.evk, galois, o))
        return o.reshape(P.dnum, 2, P.n_q + P.n_p, P.n)

    def pk_words(self):
        P = self.params
        o = np.zeros(2 * P.n_q * P.n, np.uint64)
        check(L.hs_public_key_export(self.pk, o))
        return o.reshape(2, P.n_q, P.n)

    def decrypt(self, words):
        """words: ncomp x (level+1) x N (e.g. Ciphertext.words()) -> coefficient residues"""
        words = np.ascontiguousarray(words, np.uint64)
        nc, l1, n = words.shape
        o = np.zeros(l1 * n, np.uint64)
        check(L.hs_ckks_decrypt_host(self.sk, words.ravel(), l1 - 1, nc, o))
        return o.reshape(l1, n)

    def decrypt_decode(self, ct, level_scale=None):
        w = ct.words() if hasattr(ct, "words") else ct
        m = self.decrypt(w)
        level = m.shape[0] - 1
        return self.params.decode(m[0], self.params.scale(level) if level_scale is None else level_scale)


class Ciphertext:
    def __init__(self, ctx: Context, ptr, owner=None):
        # owner: the object that owns a borrowed handle (a Plan's outputs)
        self.ctx, self.ptr, self.owner = ctx, ptr, owner

    def __del__(self):
        if getattr(self, "ptr", None) and self.owner is None:
            L.hs_ct_destroy(self.ptr)
            self.ptr = None

    @property
    def level(self):
        return L.hs_ct_level(self.ptr)

    @property
    def ncomp(self):
        return L.hs_ct_ncomp(self.ptr)

    @property
    def scale(self):
        """declared encoding scale, else the canonical scale of its level (C11)"""
        return float(L.hs_ct_scale(self.ptr))

    def set_scale(self, scale):
        """hs_ct_set_scale: declare the scale this ciphertext was encoded at"""
        check(L.hs_ct_set_scale(self.ptr, float(scale)))
        return self

    def words(self, stream=None):
        P = self.ctx.params
        w = np.zeros(self.ncomp * (self.level + 1) * P.n, np.uint64)
        check(L.hs_ct_export(self.ctx.ptr, self.ptr, w.ctypes.data_as(C.c_void_p), 0, _stream(stream)))
        return w.reshape(self.ncomp, self.level + 1, P.n)

    @classmethod
    def from_words(cls, ctx, words, stream=None):
        words = np.ascontiguousarray(words, np.uint64)
        nc, l1, _ = words.shape
        out = C.c_void_p()
        check(L.hs_ct_import(ctx.ptr, l1 - 1, nc, words.ctypes.data_as(C.c_void_p), 0, _stream(stream),
                             C.byref(out)))
        return cls(ctx, out)


def encrypt(keys: Keys, pt, level, seed, idx, use_sk=False, stream=None) -> Ciphertext:
    out = C.c_void_p()
    check(L.hs_ckks_encrypt(keys.ctx.ptr, keys.ptr, np.ascontiguousarray(pt, np.uint64).ravel(), level, seed, idx,
                            1 if use_sk else 0, _stream(stream), C.byref(out)))
    return Ciphertext(keys.ctx, out)


def decrypt(keys: Keys, ct: Ciphertext, stream=None):
    P = keys.ctx.params
    o = np.zeros((ct.level + 1) * P.n, np.uint64)
    check(L.hs_ckks_decrypt(keys.ctx.ptr, keys.ptr, ct.ptr, o, _stream(stream)))
    return o.reshape(ct.level + 1, P.n)


def decrypt_decode(keys: Keys, ct: Ciphertext, stream=None):
    P = keys.ctx.params
    m = decrypt(keys, ct, stream)
    return P.decode(m[0], P.scale(ct.level))


def op(keys, name, a: Ciphertext, b: Ciphertext = None, c=0.0, i=0, stream=None) -> Ciphertext:
    ctx = a.ctx
    out = C.c_void_p()
    check(L.hs_op(ctx.ptr, keys.ptr if keys is not None else None, L.OPS[name], a.ptr,
                  b.ptr if b is not None else None, float(c), int(i), _stream(stream), C.byref(out)))
    return Ciphertext(ctx, out)


def mult_pt(a: Ciphertext, re, im=None, target=None, stream=None) -> Ciphertext:
    re = np.ascontiguousarray(re, np.float64)
    imp = None if im is None else np.ascontiguousarray(im, np.float64)
    out = C.c_void_p()
    check(L.hs_mult_pt(a.ctx.ptr, a.ptr, re, None if imp is None else imp.ctypes.data_as(C.c_void_p),
                       a.level - 1 if target is None else target, _stream(stream), C.byref(out)))
    return Ciphertext(a.ctx, out)


def keyswitch(keys: Keys, galois, level, d_ptr, out0_ptr, out1_ptr, stream=None):
    check(L.hs_keyswitch(keys.ctx.ptr, keys.ptr, galois, level, C.c_void_p(d_ptr), C.c_void_p(out0_ptr),
                         C.c_void_p(out1_ptr), _stream(stream)))


def keyswitch_partial(keys: Keys, galois, level, d_ptr, digit_begin, digit_end, acc_ptr, stream=None):
    """hs_keyswitch_partial: the C7 accumulator of digits [digit_begin, digit_end)."""
    check(L.hs_keyswitch_partial(keys.ctx.ptr, keys.ptr, galois, level, C.c_void_p(d_ptr), digit_begin, digit_end,
                                 C.c_void_p(acc_ptr), _stream(stream)))


def ks_acc_add(ctx: Context, level, acc_ptr, other_ptr, stream=None):
    check(L.hs_ks_acc_add(ctx.ptr, level, C.c_void_p(acc_ptr), C.c_void_p(other_ptr), _stream(stream)))


def keyswitch_finish(ctx: Context, level, acc_ptr, out0_ptr, out1_ptr, stream=None):
    check(L.hs_keyswitch_finish(ctx.ptr, level, C.c_void_p(acc_ptr), C.c_void_p(out0_ptr), C.c_void_p(out1_ptr),
                                _stream(stream)))


def keyswitch_sharded(keys: Keys, galois, level, d_ptr, rank, world, out0_ptr, out1_ptr, comm=None, exchange=None,
                      stream=None):
    """hs_keyswitch_sharded: this rank's digit share, all-gather, modular sum, ModDown."""
    fn = L.EXCHANGE_FN(0) if exchange is None else exchange
    check(L.hs_keyswitch_sharded(keys.ctx.ptr, keys.ptr, galois, level, C.c_void_p(d_ptr), rank, world,
                                 comm.ptr if comm is not None else None, fn, None, C.c_void_p(out0_ptr),
                                 C.c_void_p(out1_ptr), _stream(stream)))


def gather(cts, stream=None) -> Ciphertext:
    """hs_ct_gather: one batch handle over ciphertexts of one level; hs ops on it
    run every kernel once over all members."""
    ptrs = (C.c_void_p * len(cts))(*[c.ptr.value if isinstance(c.ptr, C.c_void_p) else c.ptr for c in cts])
    out = C.c_void_p()
    check(L.hs_ct_gather(cts[0].ctx.ptr, ptrs, len(cts), _stream(stream), C.byref(out)))
    return Ciphertext(cts[0].ctx, out)


def member(batch: Ciphertext, i, stream=None) -> Ciphertext:
    out = C.c_void_p()
    check(L.hs_ct_member(batch.ctx.ptr, batch.ptr, i, _stream(stream), C.byref(out)))
    return Ciphertext(batch.ctx, out)


def rotate_hoisted(keys: Keys, a: Ciphertext, rots, stream=None):
    """C16: Rot(a, r) for every r in rots from ONE ModUp of a's c1."""
    r = (C.c_int32 * len(rots))(*rots)
    out = (C.c_void_p * len(rots))()
    check(L.hs_rotate_hoisted(keys.ctx.ptr, keys.ptr, a.ptr, r, len(rots), _stream(stream), out))
    return [Ciphertext(a.ctx, C.c_void_p(out[i])) for i in range(len(rots))]


def _poly(p):
    c = np.ascontiguousarray(p["coeffs"], np.float64)
    return L.Poly(len(c) - 1, float(p["a"]), float(p["b"]), c.ctypes.data_as(C.POINTER(C.c_double))), c


def cheb(keys: Keys, x: Ciphertext, poly, stream=None, gain: float = 1.0) -> Ciphertext:
    """hs_cheb: x holds alpha x (alpha = 2/(b-a), G28); returns gain * p(x)."""
    pp, keep = _poly(poly)
    out = C.c_void_p()
    check(L.hs_cheb(keys.ctx.ptr, keys.ptr, x.ptr, C.byref(pp), float(gain), _stream(stream), C.byref(out)))
    return Ciphertext(x.ctx, out)


def softmax_encrypt_input(keys: Keys, slots, level: int, exp_poly, seed: int, idx: int, stream=None) -> Ciphertext:
    """hs_softmax_encrypt_input: one packed slot vector -> the Softmax input
    ciphertext at `level` (G28: encoded at level+1, public-key encrypted, one
    rescale)."""
    d, keep = _softmax_desc(1, 1, 1, 0, exp_poly, [exp_poly])
    out = C.c_void_p()
    check(L.hs_softmax_encrypt_input(keys.ctx.ptr, keys.ptr, C.byref(d), np.ascontiguousarray(slots, np.float64),
                                     int(level), seed, idx, _stream(stream), C.byref(out)))
    return Ciphertext(keys.ctx, out)


def softmax_input_level(params: Params, n, m, k, variant, exp_poly, inv_polys, world=1, bts_out_level=-1) -> int:
    """hs_softmax_input_level: the planner's cheapest input level."""
    d, keep = _softmax_desc(n, m, k, variant, exp_poly, inv_polys, world, 0)
    lv = C.c_int()
    check(L.hs_softmax_input_level(params.ptr, C.byref(d), m // world, int(bts_out_level), C.byref(lv)))
    return lv.value


def softmax_input_scale(params: Params, exp_poly, level: int) -> float:
    """hs_softmax_input_scale: the scale the Softmax inputs are encoded at
    (Delta_level * 2/(b-a) of the exp table, G28)."""
    d, keep = _softmax_desc(1, 1, 1, 0, exp_poly, [exp_poly])
    v = float(L.hs_softmax_input_scale(params.ptr, C.byref(d), int(level)))
    if v <= 0.0:
        raise ValueError("softmax_input_scale: bad level or polynomial")
    return v


def cheb_depth(deg):
    return int(L.hs_cheb_depth(deg))


class Bts:
    """hs_bts: real-slot bootstrapping plan (G11).

    cfg: a preset's "bts" entry {n_cts, n_stc, arcsine, out_level};
    table: the EvalMod cosine table {K, r, coeffs} (data/bts_tables.json)."""

    def __init__(self, ctx: Context, cfg: dict, table: dict):
        self.ctx = ctx
        pp, self._c = _poly(table)
        self._p = pp
        d = L.BtsDesc(int(table["K"]), int(table["r"]), C.pointer(self._p), int(cfg["out_level"]),
                      int(cfg["n_cts"]), int(cfg["n_stc"]), 1 if cfg["arcsine"] else 0)
        out = C.c_void_p()
        check(L.hs_bts_create(ctx.ptr, C.byref(d), C.byref(out)))
        self.ptr = out

    def __del__(self):
        if getattr(self, "ptr", None):
            L.hs_bts_destroy(self.ptr)
            self.ptr = None


def bts_rotations(params: Params, cfg: dict):
    out = np.zeros(512, np.int32)
    n = L.hs_bts_rotations(params.ptr, int(cfg["n_cts"]), int(cfg["n_stc"]), out, 512)
    return [int(v) for v in out[:n]]


def bts_exponent(params: Params, arcsine: bool, bound: float) -> int:
    return int(L.hs_bts_exponent(params.ptr, 1 if arcsine else 0, bound))


def bootstrap(keys: Keys, bts: Bts, ct: Ciphertext, bound=1.0, stream=None) -> Ciphertext:
    out = C.c_void_p()
    check(L.hs_bootstrap(keys.ctx.ptr, keys.ptr, bts.ptr, ct.ptr, float(bound), _stream(stream), C.byref(out)))
    return Ciphertext(keys.ctx, out)


def variant_code(variant):
    """"A" / 0: Alg 1; "B" / 1: version B; "S" / 2: square-and-normalize (G26);
    "T3" / 3: cube-and-normalize (App. C, G27)."""
    codes = {"A": 0, "B": 1, "S": 2, "T3": 3, 0: 0, 1: 1, 2: 2, 3: 3}
    if variant not in codes:
        raise ValueError(f"unknown Softmax variant {variant!r}")
    return codes[variant]


class Comm:
    """hs_comm_init: a library-owned NCCL communicator.
    uid: the 128 bytes of Comm.unique_id() from rank 0, broadcast by the caller."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(L.hs_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx, rank, world, uid: bytes):
        assert len(uid) == 128
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        p = C.c_void_p()
        check(L.hs_comm_init(ctx.ptr, rank, world, buf, C.byref(p)))
        self.ptr, self.rank, self.world, self.ctx = p, rank, world, ctx

    def __del__(self):
        if getattr(self, "ptr", None):
            L.hs_comm_destroy(self.ptr)
            self.ptr = None


def _softmax_desc(n, m, k, variant, exp_poly, inv_polys, world=1, rank=0, exchange=None, bts=None, comm=None,
                  aux_split=0):
    keep = []
    e, c = _poly(exp_poly)
    keep.append(c)
    arr = (L.Poly * len(inv_polys))()
    for i, p in enumerate(inv_polys):
        pp, c = _poly(p)
        keep.append(c)
        arr[i] = pp
    ep = (L.Poly * 1)(e)
    keep += [arr, ep]
    fn = L.EXCHANGE_FN(0) if exchange is None else exchange
    keep.append(fn)
    # a table's last entry may carry "newton": the polynomial is then a seed (G24)
    d = L.SoftmaxDesc(n, m, k, variant_code(variant), ep, arr, world, rank, fn, None,
                      bts.ptr if bts is not None else None, int(inv_polys[-1].get("newton", 0)),
                      comm.ptr if comm is not None else None, int(aux_split))
    keep.append(comm)
    return d, keep


def softmax_one_ctxt(keys: Keys, ct: Ciphertext, n, k, variant, exp_poly, inv_polys, bts=None,
                     stream=None) -> Ciphertext:
    d, keep = _softmax_desc(n, 1, k, variant, exp_poly, inv_polys, bts=bts)
    out = C.c_void_p()
    check(L.hs_softmax_one_ctxt(keys.ctx.ptr, keys.ptr, C.byref(d), ct.ptr, _stream(stream), C.byref(out)))
    return Ciphertext(keys.ctx, out)


def _sched_dict(s):
    return {f: getattr(s, f) for f, _ in L.SoftmaxSched._fields_}


def softmax_schedule(params: Params, n, m, k, variant, exp_poly, inv_polys, in_level, m_local=None, world=1,
                     bts_out_level=-1) -> dict:
    """hs_softmax_schedule: the Softmax driver's schedule planned on the host
    (no device, no keys): output level, main / aux bootstraps, products,
    rotations and the modelled cost."""
    d, keep = _softmax_desc(n, m, k, variant, exp_poly, inv_polys, world, 0)
    s = L.SoftmaxSched()
    ml = m // world if m_local is None else m_local
    check(L.hs_softmax_schedule(params.ptr, C.byref(d), int(in_level), ml, int(bts_out_level), C.byref(s)))
    return _sched_dict(s)


def softmax_choose(params: Params, candidates, n, m, in_level, world=1, bts_out_level=-1):
    """hs_softmax_choose: automatic variant selection.  candidates: list of
    dicts {k, variant, exp, inv} (a poly_tables.json entry plus its k and
    variant).  Returns (index of the cheapest plan that fits, [plans])."""
    descs = (L.SoftmaxDesc * len(candidates))()
    keep = []
    for i, c in enumerate(candidates):
        d, kp = _softmax_desc(n, m, c["k"], c["variant"], c["exp"], c["inv"], world, 0)
        descs[i] = d
        keep.append(kp)
    sched = (L.SoftmaxSched * len(candidates))()
    best = C.c_size_t()
    check(L.hs_softmax_choose(params.ptr, descs, len(candidates), int(in_level), m // world, int(bts_out_level),
                              C.byref(best), sched))
    return best.value, [_sched_dict(s) for s in sched]


class Plan:
    """hs_softmax_plan_create: one single-GPU Softmax captured as a CUDA graph,
    bound to the input ciphertexts `cts` (re-read at every run); outputs are
    plan-owned and overwritten by each run()."""

    def __init__(self, keys: Keys, cts, n, m, k, variant, exp_poly, inv_polys, bts=None, stream=None, comm=None,
                 aux_split=0):
        """comm: a Comm of world > 1 makes this a sharded plan (this rank's
        m / world ciphertexts; the NCCL all-gather is captured in the graph).
        aux_split: digit-split the aux thread's key switches (hs_softmax_desc)."""
        # the captured graph bakes in device pointers of the keys, the input
        # ciphertexts, the bootstrapping plan's transforms and the communicator:
        # the plan keeps every one of them alive
        self.keys, self.cts, self._bts, self._comm = keys, list(cts), bts, comm
        world, rank = (comm.world, comm.rank) if comm is not None else (1, 0)
        self._d, self._keep = _softmax_desc(n, m, k, variant, exp_poly, inv_polys, world, rank, None, bts, comm,
                                            aux_split)
        ml = len(cts)
        ins = (C.c_void_p * ml)(*[c.ptr.value if isinstance(c.ptr, C.c_void_p) else c.ptr for c in cts])
        p = C.c_void_p()
        check(L.hs_softmax_plan_create(keys.ctx.ptr, keys.ptr, C.byref(self._d), ins, ml, _stream(stream),
                                       C.byref(p)))
        self.ptr = p
        self.outputs = [Ciphertext(keys.ctx, C.c_void_p(L.hs_plan_output(p, i)), owner=self) for i in range(ml)]

    def run(self, stream=None):
        check(L.hs_plan_run(self.ptr, _stream(stream)))
        return self.outputs

    def __del__(self):
        if getattr(self, "ptr", None):
            L.hs_plan_destroy(self.ptr)
            self.ptr = None


def softmax_many_ctxt(keys: Keys, cts, n, m, k, variant, exp_poly, inv_polys, world=1, rank=0, exchange=None,
                      bts=None, stream=None, comm=None, aux_split=0):
    """cts: this rank's m/world ciphertexts.  world > 1 needs comm (a Comm,
    native NCCL) or exchange (an EXCHANGE_FN, see paper_2410_11184_b200.dist).
    aux_split: digit-split the aux thread's key switches over the ranks (1),
    or emulate that split over G ranks in this process (G >= 2, world 1)."""
    if comm is not None:
        world, rank = comm.world, comm.rank
    d, keep = _softmax_desc(n, m, k, variant, exp_poly, inv_polys, world, rank, exchange, bts, comm, aux_split)
    ml = len(cts)
    ins = (C.c_void_p * ml)(*[c.ptr.value if isinstance(c.ptr, C.c_void_p) else c.ptr for c in cts])
    outs = (C.c_void_p * ml)()
    check(L.hs_softmax_many_ctxt(keys.ctx.ptr, keys.ptr, C.byref(d), ins, ml, _stream(stream), outs))
    return [Ciphertext(keys.ctx, C.c_void_p(outs[i])) for i in range(ml)]
