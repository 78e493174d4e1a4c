"""Where does a config-3 step go?  (dev tool, GPU)  Times the whole step, one
bootstrap at the aux-thread input level, and the per-class kernel totals of
one step, so the bootstrap share and the main-thread share can be read off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench


def timeit(fn, reps=3):
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
    torch.cuda.set_device(0)
    S = bench.build_setup("config3", 0, 1, 0)
    hs, K, B, tab, P = S["hs"], S["K"], S["B"], S["tab"], S["P"]

    def step():
        hs.softmax_many_ctxt(K, S["cts"], S["n"], S["m"], S["k"], S["wl"]["variant"], tab["exp"], tab["inv"], bts=B)

    t_step = timeit(step, 2)
    print(f"step {t_step:.1f} ms")
    z = np.random.default_rng(1).uniform(-1, 1, P.n // 2)
    ct0 = hs.encrypt(K, P.encode(z, scale=P.scale(0), level=0), 0, 1, 0)
    t_bts = timeit(lambda: hs.bootstrap(K, B, ct0, 1.0), 3)
    print(f"bootstrap {t_bts:.1f} ms  (x10 per step = {10 * t_bts:.0f} ms)")
    ctx = S["ctx"]
    hs._lib.hs_kprof_enable(ctx.ptr, 1)
    hs.bootstrap(K, B, ct0, 1.0)
    kp = np.zeros(3 * len(hs._lib.KPROF_CLASSES))
    hs._lib.hs_kprof_collect(ctx.ptr, kp, len(hs._lib.KPROF_CLASSES))
    hs._lib.hs_kprof_enable(ctx.ptr, 0)
    for i, nm in enumerate(hs._lib.KPROF_CLASSES):
        if kp[3 * i]:
            print(f"  bts {nm:10s} {kp[3 * i + 1]:8.2f} ms  {int(kp[3 * i])} launches")
    for lvl in [12, 8, 4]:
        ct = hs.encrypt(K, P.encode(z, scale=P.scale(lvl), level=lvl), lvl, 1, 0)
        t = timeit(lambda: hs.op(K, "mult", ct, ct), 10)
        print(f"HMult level {lvl}: {t * 1e3:.0f} us")


if __name__ == "__main__":
    main()
