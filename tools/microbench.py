"""Primitive micro-benchmarks on the GPU (dev tool): NTT per limb, key switch,
HMult+relin+rescale and rotation at N = 2^16 user levels, CUDA-event timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_11184_b200 as hs
import workloads as W


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    pre = W.preset("P16")
    P = hs.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    K = hs.Keys(ctx, 1, pre["h"], galois=[P.galois_of_rot(1)])
    n_limbs = 32
    data = torch.randint(0, 2 ** 40, (n_limbs * P.n,), dtype=torch.int64, device="cuda")
    t = timeit(lambda: ctx.ntt(data.data_ptr(), 0, n_limbs))
    print(f"NTT fwd: {t * 1e3 / n_limbs:.2f} us/limb ({n_limbs} limbs/launch)")
    t = timeit(lambda: ctx.ntt(data.data_ptr(), 0, n_limbs, inverse=True))
    print(f"NTT inv: {t * 1e3 / n_limbs:.2f} us/limb")
    z = np.random.default_rng(0).uniform(-1, 1, P.n // 2)
    for lvl in [12, 6, 28]:
        ct = hs.encrypt(K, P.encode(z, scale=P.scale(lvl), level=lvl), lvl, 1, 0)
        t = timeit(lambda: hs.op(K, "mult", ct, ct), 10)
        tr = timeit(lambda: hs.op(K, "rotate", ct, i=1), 10)
        print(f"level {lvl}: HMult+relin+rescale {t * 1e3:.1f} us, rotation {tr * 1e3:.1f} us")
    hs._lib.hs_kprof_enable(ctx.ptr, 1)
    ct = hs.encrypt(K, P.encode(z, scale=P.scale(12), level=12), 12, 1, 0)
    for _ in range(10):
        hs.op(K, "mult", ct, ct)
    kp = np.zeros(3 * len(hs._lib.KPROF_CLASSES))
    hs._lib.hs_kprof_collect(ctx.ptr, kp, len(hs._lib.KPROF_CLASSES))
    for i, nm in enumerate(hs._lib.KPROF_CLASSES):
        if kp[3 * i]:
            print(f"  {nm:10s} {kp[3 * i + 1] / 10 * 1e3:8.1f} us/HMult  {kp[3 * i + 2] / kp[3 * i + 1] / 1e6:8.1f} GB/s"
                  f"  ({int(kp[3 * i] / 10)} launches)")


if __name__ == "__main__":
    main()
