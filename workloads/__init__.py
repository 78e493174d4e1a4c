"""Seeded synthetic inputs and parameter presets shared by the tests, the
oracle harness and bench.py.

This module holds NO arithmetic of the method: only parameter *data*
(prime bit sizes, anchors), the synthetic input distribution of the paper's
experiments (PAPER.md 466-475: x ~ N(-M/2, (M/6)^2) tail-cut to [-M, 0] by
resampling, G17) and the seed derivation.  Both the CUDA path and
the oracle consume what it produces; neither imports the other.
"""
from __future__ import annotations

import json
import os

import numpy as np

BASE_SEED = 0x241011184
_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "data")


def _anchors(n_q, pairs):
    a = [0] * n_q
    for lvl, v in pairs:
        a[lvl] = v
    return a


# Parameter presets.  q_bits[l] is the bit size of
# q_l (level l), p_bits the special primes; log2_anchor[l] != 0 pins the
# canonical scale of level l to 2^anchor (C12), 0 = derived by Delta^2/q.
PRESETS = {
    # tiny ring for big-integer pins of the oracle (N = 32, insecure)
    "TINY": dict(log_n=5, q_bits=[60, 40, 40, 40], p_bits=[61], alpha=1,
                 log2_anchor=_anchors(4, [(3, 40)]), h=8),
    # config 1: N = 2^12, 12 Q limbs (exp 3 + aux 1 + 4 + 1 + main 2 =
    # 11 levels with level-exact polynomials, C13/G28), 2 special primes
    # (alpha = 2), no BTS (insecure toy)
    "TOY12": dict(log_n=12, q_bits=[60] + [40] * 11, p_bits=[61, 61], alpha=2,
                  log2_anchor=_anchors(12, [(11, 40)]), h=192),
    # N = 2^12 with a deep chain (28 Q limbs): toy Softmax with k = 2 (parity only)
    "TOY12D": dict(log_n=12, q_bits=[60] + [40] * 27, p_bits=[61, 61, 61], alpha=3,
                   log2_anchor=_anchors(28, [(27, 40)]), h=192),
    # configs 2-5: N = 2^16, FGb-shaped.  Levels: 0 (60b), 1-13 user (42b, Delta=2^42:
    # at N = 2^16 a fresh encryption's slot noise is ~2^-20.4 at Delta = 2^40 and
    # bounds everything downstream; the 13th user
    # level lets version B's fourth aux iteration -- x^-1/2^4 (5 levels),
    # lambda lambda_j and the mask from a fresh bootstrap -- stay above the 6
    # levels its main update needs: 7 instead of 8 bootstraps for config 3),
    # 14-16 SlotToCoeff (48b), 17-27 EvalMod + arcsine (~2^59: cosine series 6
    # levels with the level-exact C13, 3 double angles, arcsine 2),
    # 28-31 CoeffToSlot (60b); 5 special primes of 61 bits (alpha = 5, dnum = 7).
    "P16": dict(log_n=16, q_bits=[60] + [42] * 13 + [48] * 3 + [59] * 11 + [60] * 4, p_bits=[61] * 5, alpha=5,
                log2_anchor=_anchors(32, [(31, 60), (30, 63), (29, 62), (28, 60), (27, 59), (15, 48), (14, 48),
                                          (13, 42)]),
                h=192, bts=dict(table="K24_r3_d63", n_cts=4, n_stc=3, arcsine=True, out_level=13)),
    # N = 2^16 with only the user chain (levels 0-12): primitive parity and
    # key-switch measurements at the user levels without BTS-sized keys.
    "P16U": dict(log_n=16, q_bits=[60] + [42] * 13, p_bits=[61] * 5, alpha=5,
                 log2_anchor=_anchors(14, [(13, 42)]), h=192),
}


def preset(name: str) -> dict:
    return dict(PRESETS[name])


def derive_seed(*parts) -> int:
    """Deterministic 64-bit seed from the base seed and a tag path (SplitMix64)."""
    x = BASE_SEED
    for p in parts:
        v = p if isinstance(p, int) else int.from_bytes(str(p).encode()[:8].ljust(8, b"\0"), "little")
        x = (x ^ v) & 0xFFFFFFFFFFFFFFFF
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        x = z ^ (z >> 31)
    return x


def softmax_inputs(L: int, n: int, M: float, seed: int, dist: str = "normal") -> np.ndarray:
    """L Softmax inputs of dimension n in [-M, 0] (PAPER.md 466-475)."""
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        return rng.uniform(-M, 0.0, size=(L, n))
    x = rng.normal(-M / 2, M / 6, size=(L, n))
    bad = (x < -M) | (x > 0)
    while bad.any():
        x[bad] = rng.normal(-M / 2, M / 6, size=int(bad.sum()))
        bad = (x < -M) | (x > 0)
    return x


def poly_tables() -> dict:
    with open(os.path.join(_DATA, "poly_tables.json")) as fh:
        return json.load(fh)


# Softmax workloads of BASELINE.json's configs
WORKLOADS = {
    "config1": dict(preset="TOY12", n=16, L=128, m=1, M=2.0, k=1, variant="A", table="toy_n16_M2_k1_A"),
    "config2": dict(preset="P16", n=256, L=128, m=1, M=128.0, k=5, variant="A", table="p16_n256_M128_k5_A"),
    # input_level: the level the inputs are encrypted at (hs_softmax_input_level's
    # pick for this workload; tests/test_schedule.py checks the two agree)
    "config3": dict(preset="P16", n=256, L=8192, m=64, M=128.0, k=5, variant="B", table="p16_n256_M128_k5_B",
                    input_level=10),
    # config 2 with the square-and-normalize variant (PAPER.md 757-765, G26)
    "config2S": dict(preset="P16", n=256, L=128, m=1, M=128.0, k=5, variant="S", table="p16_n256_M128_k5_S"),
    "config4": dict(preset="P16", n=128, L=4096, m=16, M=128.0, k=5, variant="B", table="p16_n128_M128_k5_B"),
    # one Softmax of dimension N0 = 32768 (Alg 1, k = 7; last step
    # seed + Newton, G24)
    "config5": dict(preset="P16", n=32768, L=1, m=1, M=256.0, k=7, variant="A", table="p16_n32768_M256_k7_A"),
}


def bts_tables() -> dict:
    with open(os.path.join(_DATA, "bts_tables.json")) as fh:
        return json.load(fh)


# P16 with 12 user levels (round-2 comparison point: 8 bootstraps for config 3
# instead of 7); bench.py HS_PRESET=P16L12
PRESETS["P16L12"] = dict(PRESETS["P16"], q_bits=[60] + [42] * 12 + [48] * 3 + [59] * 11 + [60] * 4,
                         log2_anchor=_anchors(31, [(30, 60), (29, 63), (28, 62), (27, 60), (26, 59), (14, 48),
                                                   (13, 48), (12, 42)]),
                         bts=dict(PRESETS["P16"]["bts"], out_level=12))

# Chains within the HE standard's 128-bit bound for N = 2^16 (log QP <= 1772,
# DESIGN.md section 4): smaller bootstrapping primes and 12 / 11 user levels.
# Measurement presets (bench.py HS_PRESET=...), not the headline chain.
PRESETS["P16S12"] = dict(PRESETS["P16"], q_bits=[60] + [42] * 12 + [46] * 3 + [49] * 11 + [57] * 4, p_bits=[60] * 5,
                         log2_anchor=_anchors(31, [(30, 57), (29, 60), (28, 59), (27, 57), (26, 49), (14, 46),
                                                   (13, 46), (12, 42)]),
                         bts=dict(PRESETS["P16"]["bts"], out_level=12))
PRESETS["P16S11"] = dict(PRESETS["P16"], q_bits=[60] + [42] * 11 + [46] * 3 + [53] * 11 + [57] * 4, p_bits=[60] * 5,
                         log2_anchor=_anchors(30, [(29, 57), (28, 60), (27, 59), (26, 57), (25, 53), (13, 46),
                                                   (12, 46), (11, 42)]),
                         bts=dict(PRESETS["P16"]["bts"], out_level=11))

# N = 2^12 ring with P16's exact modulus chain (bootstrapping included):
# parity / precision tests of configs 2-5 at a size the oracle finishes quickly.
PRESETS["TOY12B"] = dict(PRESETS["P16"], log_n=12)
