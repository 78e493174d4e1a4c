"""Probe bootstrapping precision on the GPU at a given preset (dev tool)."""
import sys, os, math, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import workloads as W
import paper_2410_11184_b200 as hs

pre = W.preset(sys.argv[1] if len(sys.argv) > 1 else "P16")
cfg = dict(pre["bts"])
if len(sys.argv) > 2:
    cfg["table"] = sys.argv[2]
print("table", cfg["table"])
P = hs.Params.from_preset(pre)
ctx = hs.Context(P, 0)
gal = sorted({P.galois_of_rot(r) for r in hs.bts_rotations(P, cfg)} | {2 * P.n - 1})
t = time.time()
K = hs.Keys(ctx, 5, pre["h"], galois=gal)
print("keygen", round(time.time() - t, 1), "s", len(gal), "keys", flush=True)
B = hs.Bts(ctx, cfg, W.bts_tables()[cfg["table"]])
rng = np.random.default_rng(1)
for bound, kind in [(1.0, "uniform"), (1.0, "uniform"), (1.0, "const"), (1.5, "const"), (300.0, "uniform")]:
    if kind == "uniform":
        z = rng.uniform(-bound, bound, P.n // 2)
    else:
        z = np.full(P.n // 2, bound * 0.8) + rng.uniform(-0.01, 0.01, P.n // 2)
    pt = P.encode(z, scale=P.scale(3), level=3)
    ct = hs.encrypt(K, pt, 3, 9, 0)
    e_in = np.abs(hs.decrypt_decode(K, ct).real - z).max()
    print(f"   input ciphertext (fresh, level 3) error 2^{math.log2(e_in):.2f}", flush=True)
    import torch; torch.cuda.synchronize()
    t = time.time()
    out = hs.bootstrap(K, B, ct, bound)
    torch.cuda.synchronize()
    dt = time.time() - t
    d = hs.decrypt_decode(K, out).real
    ea = np.abs(d - z)
    err = ea.max()
    # multiplicative part: d - z ~ eps z + residual
    eps = float(((d - z) * z).sum() / (z * z).sum())
    res = np.abs(d - z - eps * z).max()
    print(f"   gain error eps = {eps:.3e}, residual after removing it 2^{math.log2(res):.2f}", flush=True)
    pc = " ".join(f"p{q}=2^{math.log2(np.percentile(ea, q)):.1f}" for q in (50, 99, 99.99))
    print(f"bound {bound} {kind}: e={hs.bts_exponent(P, cfg['arcsine'], bound)} abs err 2^{math.log2(err):.2f} "
          f"rel 2^{math.log2(err/np.abs(z).max()):.2f} [{pc}] ({dt:.3f}s)", flush=True)
