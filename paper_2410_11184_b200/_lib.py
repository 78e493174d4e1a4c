"""Thin ctypes binding of libhesoftmax.so (include/hesoftmax.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  If the shared library is missing this module raises at import
time -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhesoftmax.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `make -C {_HERE}` or __graft_entry__.build()")

_L = C.CDLL(LIB_PATH)

vp = C.c_void_p
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

STATUS = ["HS_OK", "HS_EINVAL", "HS_ELEVEL", "HS_EKEY", "HS_ESCALE", "HS_EOVERFLOW", "HS_EDOMAIN",
          "HS_ENOMEM", "HS_ECUDA", "HS_ENCCL"]
OPS = dict(add=0, sub=1, mult=2, tensor=3, relin=4, rescale=5, level_down=6, mult_const=7, add_const=8,
           mult_int=9, rotate=10, conj=11, galois=12)
LEDGER = ["hmult", "tensor", "ks", "rot", "rescale", "cmult", "pmult", "leveldown", "bts", "ntt", "kernels",
          "ntt_fp"]


class HsError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"{STATUS[code] if 0 <= code < len(STATUS) else code}: {msg}")


class ParamsDesc(C.Structure):
    _fields_ = [("log_n", C.c_int), ("n_q", C.c_int), ("q_bits", C.POINTER(C.c_int)), ("n_p", C.c_int),
                ("p_bits", C.POINTER(C.c_int)), ("alpha", C.c_int), ("log2_anchor", C.POINTER(C.c_int))]


class Poly(C.Structure):
    _fields_ = [("deg", C.c_int), ("a", C.c_double), ("b", C.c_double), ("coeffs", C.POINTER(C.c_double))]


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, vp, vp, vp, C.c_size_t, vp)


class SoftmaxDesc(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("k", C.c_int), ("variant", C.c_int),
                ("exp_poly", C.POINTER(Poly)), ("inv_poly", C.POINTER(Poly)), ("world", C.c_int),
                ("rank", C.c_int), ("exchange", EXCHANGE_FN), ("exchange_user", vp), ("bts", vp),
                ("newton", C.c_int), ("comm", vp), ("aux_split", C.c_int)]


class SoftmaxSched(C.Structure):
    _fields_ = [("out_level", C.c_int), ("bts_main", C.c_int), ("bts_aux", C.c_int), ("hmult", C.c_int),
                ("rotations", C.c_int), ("poly_evals", C.c_int), ("exchanges", C.c_int), ("cost", C.c_double)]


class BtsDesc(C.Structure):
    _fields_ = [("K", C.c_int), ("r", C.c_int), ("cos_poly", C.POINTER(Poly)), ("out_level", C.c_int),
                ("n_cts", C.c_int), ("n_stc", C.c_int), ("arcsine", C.c_int)]


def _sig(name, res, args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = args
    return f


hs_last_error = _sig("hs_last_error", C.c_char_p, [])
hs_ckks_params = _sig("hs_ckks_params", C.c_int, [C.POINTER(ParamsDesc), C.POINTER(vp)])
hs_params_destroy = _sig("hs_params_destroy", None, [vp])
hs_params_log_n = _sig("hs_params_log_n", C.c_int, [vp])
hs_params_n_q = _sig("hs_params_n_q", C.c_int, [vp])
hs_params_n_p = _sig("hs_params_n_p", C.c_int, [vp])
hs_params_primes = _sig("hs_params_primes", C.c_int, [vp, u64p])
hs_params_psi = _sig("hs_params_psi", C.c_uint64, [vp, C.c_int])
hs_params_scale = _sig("hs_params_scale", C.c_double, [vp, C.c_int])
hs_galois_of_rot = _sig("hs_galois_of_rot", C.c_int, [vp, C.c_int])
hs_context_create = _sig("hs_context_create", C.c_int, [vp, C.c_int, C.POINTER(vp)])
ALLOC_FN = C.CFUNCTYPE(vp, C.c_size_t, vp, vp)
FREE_FN = C.CFUNCTYPE(None, vp, C.c_size_t, vp, vp)


class Allocator(C.Structure):
    """hs_allocator"""
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", vp)]


hs_context_create_ex = _sig("hs_context_create_ex", C.c_int, [vp, C.c_int, C.POINTER(Allocator), C.POINTER(vp)])
hs_context_destroy = _sig("hs_context_destroy", None, [vp])
hs_ckks_keygen = _sig("hs_ckks_keygen", C.c_int,
                      [vp, C.c_uint64, C.c_int, i32p, C.c_size_t, C.c_int, vp, C.POINTER(vp)])
hs_keys_destroy = _sig("hs_keys_destroy", None, [vp])
hs_ckks_keygen_host = _sig("hs_ckks_keygen_host", C.c_int, [vp, C.c_uint64, C.c_int, i32p, C.c_size_t, C.c_int,
                                                            C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)])
hs_keys_upload = _sig("hs_keys_upload", C.c_int, [vp, vp, vp, vp, C.POINTER(vp)])
hs_ckks_decrypt_host = _sig("hs_ckks_decrypt_host", C.c_int, [vp, u64p, C.c_int, C.c_int, u64p])
hs_secret_key_export = _sig("hs_secret_key_export", C.c_int, [vp, i64p])
hs_eval_keys_count = _sig("hs_eval_keys_count", C.c_size_t, [vp])
hs_eval_keys_export = _sig("hs_eval_keys_export", C.c_int, [vp, C.c_int, u64p])
hs_public_key_export = _sig("hs_public_key_export", C.c_int, [vp, u64p])
hs_secret_key_destroy = _sig("hs_secret_key_destroy", None, [vp])
hs_public_key_destroy = _sig("hs_public_key_destroy", None, [vp])
hs_eval_keys_destroy = _sig("hs_eval_keys_destroy", None, [vp])
hs_keys_export_swk = _sig("hs_keys_export_swk", C.c_int, [vp, vp, C.c_int, u64p])
hs_keys_export_secret = _sig("hs_keys_export_secret", C.c_int, [vp, vp, i64p])
hs_ckks_encode = _sig("hs_ckks_encode", C.c_int, [vp, f64p, vp, C.c_size_t, C.c_int, C.c_double, u64p])
hs_ckks_decode = _sig("hs_ckks_decode", C.c_int, [vp, u64p, C.c_double, f64p, f64p, C.c_size_t])
hs_pack = _sig("hs_pack", C.c_int, [f64p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, f64p])
hs_unpack = _sig("hs_unpack", C.c_int, [f64p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, f64p])
hs_ckks_encrypt = _sig("hs_ckks_encrypt", C.c_int,
                       [vp, vp, u64p, C.c_int, C.c_uint64, C.c_uint64, C.c_int, vp, C.POINTER(vp)])
hs_ckks_decrypt = _sig("hs_ckks_decrypt", C.c_int, [vp, vp, vp, u64p, vp])
hs_ct_import = _sig("hs_ct_import", C.c_int, [vp, C.c_int, C.c_int, vp, C.c_int, vp, C.POINTER(vp)])
hs_ct_export = _sig("hs_ct_export", C.c_int, [vp, vp, vp, C.c_int, vp])
hs_ct_level = _sig("hs_ct_level", C.c_int, [vp])
hs_ct_set_scale = _sig("hs_ct_set_scale", C.c_int, [vp, C.c_double])
hs_ct_scale = _sig("hs_ct_scale", C.c_double, [vp])
hs_ctx_debug_domain = _sig("hs_ctx_debug_domain", C.c_int, [vp, vp])
hs_ct_ncomp = _sig("hs_ct_ncomp", C.c_int, [vp])
hs_ct_destroy = _sig("hs_ct_destroy", None, [vp])
hs_ct_write = _sig("hs_ct_write", C.c_int, [vp, vp, vp, C.c_int, vp])
hs_ct_gather = _sig("hs_ct_gather", C.c_int, [vp, C.POINTER(vp), C.c_int, vp, C.POINTER(vp)])
hs_ct_batch = _sig("hs_ct_batch", C.c_int, [vp])
hs_ct_member = _sig("hs_ct_member", C.c_int, [vp, vp, C.c_int, vp, C.POINTER(vp)])
hs_softmax_plan_create = _sig("hs_softmax_plan_create", C.c_int, [vp, vp, vp, C.POINTER(vp), C.c_size_t, vp,
                                                                  C.POINTER(vp)])
hs_plan_run = _sig("hs_plan_run", C.c_int, [vp, vp])
hs_plan_n_outputs = _sig("hs_plan_n_outputs", C.c_size_t, [vp])
hs_plan_output = _sig("hs_plan_output", vp, [vp, C.c_size_t])
hs_plan_destroy = _sig("hs_plan_destroy", None, [vp])
hs_op = _sig("hs_op", C.c_int, [vp, vp, C.c_int, vp, vp, C.c_double, C.c_int, vp, C.POINTER(vp)])
hs_mult_pt = _sig("hs_mult_pt", C.c_int, [vp, vp, f64p, vp, C.c_int, vp, C.POINTER(vp)])
hs_keyswitch = _sig("hs_keyswitch", C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp, vp, vp])
hs_rotate_hoisted = _sig("hs_rotate_hoisted", C.c_int, [vp, vp, vp, C.POINTER(C.c_int32), C.c_int, vp,
                                                        C.POINTER(vp)])
hs_ntt = _sig("hs_ntt", C.c_int, [vp, C.c_int, C.c_int, vp, C.c_int, vp])
hs_keyswitch_partial = _sig("hs_keyswitch_partial", C.c_int,
                            [vp, vp, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, vp])
hs_ks_acc_add = _sig("hs_ks_acc_add", C.c_int, [vp, C.c_int, vp, vp, vp])
hs_keyswitch_finish = _sig("hs_keyswitch_finish", C.c_int, [vp, C.c_int, vp, vp, vp, vp])
hs_keyswitch_sharded = _sig("hs_keyswitch_sharded", C.c_int,
                            [vp, vp, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, EXCHANGE_FN, vp, vp, vp, vp])
hs_cheb = _sig("hs_cheb", C.c_int, [vp, vp, vp, C.POINTER(Poly), C.c_double, vp, C.POINTER(vp)])
hs_cheb_depth = _sig("hs_cheb_depth", C.c_int, [C.c_int])
hs_softmax_encrypt_input = _sig("hs_softmax_encrypt_input", C.c_int,
                                [vp, vp, C.POINTER(SoftmaxDesc), f64p, C.c_int, C.c_uint64, C.c_uint64, vp,
                                 C.POINTER(vp)])
hs_softmax_input_level = _sig("hs_softmax_input_level", C.c_int,
                              [vp, C.POINTER(SoftmaxDesc), C.c_size_t, C.c_int, C.POINTER(C.c_int)])
hs_softmax_input_scale = _sig("hs_softmax_input_scale", C.c_double, [vp, C.POINTER(SoftmaxDesc), C.c_int])
hs_softmax_one_ctxt = _sig("hs_softmax_one_ctxt", C.c_int,
                           [vp, vp, C.POINTER(SoftmaxDesc), vp, vp, C.POINTER(vp)])
hs_softmax_many_ctxt = _sig("hs_softmax_many_ctxt", C.c_int,
                            [vp, vp, C.POINTER(SoftmaxDesc), C.POINTER(vp), C.c_size_t, vp, C.POINTER(vp)])
hs_softmax_schedule = _sig("hs_softmax_schedule", C.c_int, [vp, C.POINTER(SoftmaxDesc), C.c_int, C.c_size_t,
                                                            C.c_int, C.POINTER(SoftmaxSched)])
hs_softmax_choose = _sig("hs_softmax_choose", C.c_int, [vp, C.POINTER(SoftmaxDesc), C.c_size_t, C.c_int, C.c_size_t,
                                                        C.c_int, C.POINTER(C.c_size_t), C.POINTER(SoftmaxSched)])
hs_comm_unique_id = _sig("hs_comm_unique_id", C.c_int, [C.POINTER(C.c_uint8)])
hs_comm_init = _sig("hs_comm_init", C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(vp)])
hs_comm_destroy = _sig("hs_comm_destroy", None, [vp])
hs_bts_create = _sig("hs_bts_create", C.c_int, [vp, C.POINTER(BtsDesc), C.POINTER(vp)])
hs_bts_destroy = _sig("hs_bts_destroy", None, [vp])
hs_bts_rotations = _sig("hs_bts_rotations", C.c_int, [vp, C.c_int, C.c_int, i32p, C.c_int])
hs_bts_exponent = _sig("hs_bts_exponent", C.c_int, [vp, C.c_int, C.c_double])
hs_bootstrap = _sig("hs_bootstrap", C.c_int, [vp, vp, vp, vp, C.c_double, vp, C.POINTER(vp)])
hs_ledger_get = _sig("hs_ledger_get", C.c_int, [vp, C.POINTER(C.c_int64), C.c_int])
hs_ledger_reset = _sig("hs_ledger_reset", C.c_int, [vp])

# every symbol include/hesoftmax.h declares (checked by tests/test_abi.py)
EXPORTED = [n for n in list(globals()) if n.startswith("hs_")]


def check(rc):
    if rc != 0:
        raise HsError(rc, hs_last_error().decode())

hs_kprof_enable = _sig("hs_kprof_enable", C.c_int, [vp, C.c_int])
hs_kprof_collect = _sig("hs_kprof_collect", C.c_int, [vp, np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS"),
                                                      C.c_int])
KPROF_CLASSES = ["ntt", "add", "scalar", "ptmul", "tensor", "permute", "rescale", "bconv", "ks_inner", "moddown",
                 "rng", "modraise", "ks_hoist"]
EXPORTED = [n for n in list(globals()) if n.startswith("hs_")]
