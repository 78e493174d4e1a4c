"""Where does one EvalMod Chebyshev evaluation go?  (dev tool, GPU)
Evaluates the BTS cosine series (degree 63) on one ciphertext at the level
EvalMod starts from, with per-kernel CUDA events, and prints the ledger and
kernel classes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_11184_b200 as hs
import workloads as W


def main():
    pre = W.preset("P16")
    P = hs.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    K = hs.Keys(ctx, 3, pre["h"], galois=[])
    tab = W.bts_tables()[pre["bts"]["table"]]
    lvl = 27
    z = np.random.default_rng(0).uniform(-1, 1, P.n // 2)
    ct = hs.encrypt(K, P.encode(z, scale=P.scale(lvl), level=lvl), lvl, 1, 0)
    for _ in range(2):
        hs.cheb(K, ct, tab)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.ledger_reset()
    e0.record()
    out = hs.cheb(K, ct, tab)
    e1.record()
    torch.cuda.synchronize()
    print(f"cheb deg {len(tab['coeffs']) - 1} from level {lvl} -> {out.level}: {e0.elapsed_time(e1):.2f} ms")
    print("ledger", ctx.ledger())
    hs._lib.hs_kprof_enable(ctx.ptr, 1)
    hs.cheb(K, ct, tab)
    kp = np.zeros(3 * len(hs._lib.KPROF_CLASSES))
    hs._lib.hs_kprof_collect(ctx.ptr, kp, len(hs._lib.KPROF_CLASSES))
    for i, nm in enumerate(hs._lib.KPROF_CLASSES):
        if kp[3 * i]:
            print(f"  {nm:10s} {kp[3 * i + 1]:8.3f} ms  {int(kp[3 * i])} launches")


if __name__ == "__main__":
    main()
