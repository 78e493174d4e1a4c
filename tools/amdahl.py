"""Aux / main split of the config-3 step (GPU; DESIGN.md section 7 Amdahl
table).  Version B with m = 8, 16, 32, 64 main ciphertexts (same tables,
the same aux schedule -- the planner's bootstrap count does not depend on m)
replayed as CUDA-graph plans: step(m) = T_aux + m t_main, fitted by least
squares; plus one bootstrap timed alone.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402


def timeit(fn, reps):
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
    import paper_2410_11184_b200 as hs
    torch.cuda.set_device(0)
    wl = W.WORKLOADS["config3"]
    tab = W.poly_tables()[wl["table"]]
    pre = W.preset(wl["preset"])
    P = hs.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    n, k = wl["n"], wl["k"]
    top = pre["bts"]["out_level"]
    rots = set(hs.bts_rotations(P, pre["bts"]))
    for m in (8, 16, 32, 64):
        nb = n // m
        stride = (P.n // 2) // nb
        i = 0
        while (1 << i) < nb:
            rots |= {stride << i, -(stride << i)}
            i += 1
    gal = sorted({P.galois_of_rot(r) for r in rots} | {2 * P.n - 1})
    K = hs.Keys(ctx, W.derive_seed("keys", "amdahl"), pre["h"], galois=gal)
    B = hs.Bts(ctx, pre["bts"], W.bts_tables()[pre["bts"]["table"]])
    rows = []
    for m in (8, 16, 32, 64):
        L = (P.n // 2) * m // n
        lv = hs.softmax_input_level(P, n, m, k, "B", tab["exp"], tab["inv"], 1, top)
        x = W.softmax_inputs(L, n, wl["M"], seed=m)
        slots = P.pack(x, m)
        cts = [hs.softmax_encrypt_input(K, slots[c], lv, tab["exp"], 5, c) for c in range(m)]
        plan = hs.Plan(K, cts, n, m, k, "B", tab["exp"], tab["inv"], bts=B)
        ctx.ledger_reset()
        plan.run()
        torch.cuda.synchronize()
        nbts = ctx.ledger()["bts"]
        ms = timeit(plan.run, 3)
        rows.append(dict(m=m, input_level=lv, ms=round(ms, 2), bts=nbts))
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        del plan, cts
    ms_ = np.array([r["ms"] for r in rows])
    mm = np.array([r["m"] for r in rows], float)
    A = np.stack([np.ones_like(mm), mm], 1)
    (t_aux, t_main), *_ = np.linalg.lstsq(A, ms_, rcond=None)
    z = np.random.default_rng(1).uniform(-1, 1, P.n // 2)
    ct0 = hs.encrypt(K, P.encode(z, scale=P.scale(0), level=0), 0, 1, 0)
    t_bts = timeit(lambda: hs.bootstrap(K, B, ct0, 1.0), 5)
    nb = rows[-1]["bts"]
    step = rows[-1]["ms"]
    out = dict(rows=rows, fit=dict(t_aux_ms=round(float(t_aux), 2), t_main_per_ct_ms=round(float(t_main), 3)),
               t_bts_ms=round(t_bts, 2), bts_per_step=nb, step_m64_ms=step,
               aux_fraction_m64=round(float(t_aux) / step, 3),
               bts_fraction_m64=round(nb * t_bts / step, 3))
    # strong scaling of the m = 64 step over G GPUs: main sharded by
    # ciphertext, aux replicated (the round-1 design) vs aux key switches
    # digit-split (aux_split; only the modelled key-switch share of the aux
    # work shrinks, bootstraps' hoisted / BSGS key switches stay replicated)
    proj = {}
    for G in (1, 2, 4, 8):
        proj[str(G)] = round(step / (float(t_aux) + 64 * float(t_main) / G), 2)
    out["speedup_aux_replicated"] = proj
    print(json.dumps(out))


if __name__ == "__main__":
    main()
