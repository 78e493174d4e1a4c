"""Accuracy statistics at the paper's scale (GPU; dev tool, output kept under
profiles/).

* config 2 (n = 256, M = 128, k = 5, Alg 1, one ciphertext of 128 instances):
  40 input batches = 5120 instances, as tab:alg1 (PAPER.md 494-511: 5000
  trials); worst / average / std of log2 max|error| per instance.
* config 5 (n = 32768, M = 256, k = 7, Alg 1 + Newton, G24): 5 seeds (keys,
  inputs and encryption randomness all change), worst / average bits against
  north_star's 2^-15 (the paper ran one input: -12.8 bits, PAPER.md 513-520).

usage: python tools/accuracy_stats.py [config2|config5|all] > profiles/r02_accuracy.json
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402


def setup(hs, wl, seed_tag):
    pre = W.preset(wl["preset"])
    P = hs.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    n, m = wl["n"], wl["m"]
    nb = n // m
    stride = (P.n // 2) // nb
    rots = set(hs.bts_rotations(P, pre["bts"]))
    i = 0
    while (1 << i) < nb:
        rots |= {stride << i, -(stride << i)}
        i += 1
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    K = hs.Keys(ctx, W.derive_seed("keys", seed_tag), pre["h"], galois=gal)
    B = hs.Bts(ctx, pre["bts"], W.bts_tables()[pre["bts"]["table"]])
    return pre, P, ctx, K, B


def run_batch(hs, P, K, B, wl, tab, lv, x, enc_seed):
    n, m, k = wl["n"], wl["m"], wl["k"]
    slots = P.pack(x, m)
    cts = [hs.softmax_encrypt_input(K, slots[c], lv, tab["exp"], enc_seed, c) for c in range(m)]
    out = hs.softmax_many_ctxt(K, cts, n, m, k, wl["variant"], tab["exp"], tab["inv"], bts=B)
    dec = np.stack([hs.decrypt_decode(K, c).real for c in out])
    y = P.unpack(dec, x.shape[0], n)
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    return np.log2(np.abs(y - ref).max(axis=1))


def stats(bits):
    bits = np.asarray(bits)
    return {"instances": int(bits.size), "worst_bits": round(float(bits.max()), 2),
            "avg_bits": round(float(bits.mean()), 2), "std_bits": round(float(bits.std()), 2),
            "frac_within_2^-15": round(float((bits <= -15).mean()), 5)}


def config2(hs, batches=40):
    wl = W.WORKLOADS["config2"]
    tab = W.poly_tables()[wl["table"]]
    pre, P, ctx, K, B = setup(hs, wl, "config2")
    lv = hs.softmax_input_level(P, wl["n"], wl["m"], wl["k"], wl["variant"], tab["exp"], tab["inv"], 1,
                                pre["bts"]["out_level"])
    bits = []
    t0 = time.time()
    for b in range(batches):
        x = W.softmax_inputs(wl["L"], wl["n"], wl["M"], seed=W.derive_seed("x", "config2-stats", b))
        bits.extend(run_batch(hs, P, K, B, wl, tab, lv, x, W.derive_seed("enc", "config2-stats", b)).tolist())
    return dict(workload="config2 (n=256, M=128, k=5, Alg 1, 128 instances per ciphertext)", batches=batches,
                input_level=lv, wall_s=round(time.time() - t0, 1), **stats(bits))


def config5(hs, seeds=5):
    wl = W.WORKLOADS["config5"]
    tab = W.poly_tables()[wl["table"]]
    per = []
    t0 = time.time()
    for s in range(seeds):
        pre, P, ctx, K, B = setup(hs, wl, f"config5-seed{s}")
        lv = hs.softmax_input_level(P, wl["n"], wl["m"], wl["k"], wl["variant"], tab["exp"], tab["inv"], 1,
                                    pre["bts"]["out_level"])
        x = W.softmax_inputs(wl["L"], wl["n"], wl["M"], seed=W.derive_seed("x", "config5", s))
        b = run_batch(hs, P, K, B, wl, tab, lv, x, W.derive_seed("enc", "config5", s))
        per.append(round(float(b[0]), 2))
        del K, B, ctx
    return dict(workload="config5 (n=32768, M=256, k=7, Alg 1, seed + 3 Newton steps)", seeds=seeds,
                per_seed_bits=per, worst_bits=max(per), avg_bits=round(float(np.mean(per)), 2),
                target_bits=-15, paper_bits=-12.8, wall_s=round(time.time() - t0, 1))


def main():
    import paper_2410_11184_b200 as hs
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    out = {}
    if which in ("config2", "all"):
        out["config2"] = config2(hs)
        print(json.dumps(out["config2"]), file=sys.stderr, flush=True)
    if which in ("config5", "all"):
        out["config5"] = config5(hs)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
