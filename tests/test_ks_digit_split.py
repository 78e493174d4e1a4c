"""Digit-parallel key switching ("each GPU does ModUp and
the inner product for its digit, then a modular all-reduce of 2(l+1+alpha)
limbs"), pinned on the CPU:

* single process: for every partition of the beta digits, the oracle's
  partial accumulators added mod q equal the full C7 accumulator word for
  word, and its ModDown equals the oracle's key switch (orc_keyswitch);
* world-size-2 gloo: each rank computes the accumulator of its own digits,
  the partials are all-gathered (paper_2410_11184_b200.dist.host_exchange),
  summed mod q in rank order and moved down -- every rank ends with the
  single-process key switch, bit for bit.
The product's CUDA path of the same split (hs_keyswitch_partial / _finish /
_sharded) is pinned against these words in tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

LEVEL = 9


def modsum(P, level, parts):
    primes = O.ext_primes(P, level)
    acc = np.zeros(parts[0].shape, dtype=object)
    for a in parts:
        acc = acc + a.astype(object)
    for g, q in enumerate(primes):
        acc[:, g, :] %= q
    return acc.astype(np.uint64)


def digit_ranges(beta, world):
    """rank r owns digits [r beta / world, (r + 1) beta / world)"""
    return [(r * beta // world, (r + 1) * beta // world) for r in range(world)]


def setup():
    pre = W.preset("TOY12")
    P = O.Params.from_preset(pre)
    gal = P.galois_of_rot(3)
    K = O.Keys(P, 808, pre["h"], galois=[gal])
    rng = np.random.default_rng(9)
    d = np.stack([rng.integers(0, P.primes[i], P.n, dtype=np.uint64) for i in range(LEVEL + 1)])
    return P, K, gal, d


def test_digit_partitions_sum_to_the_key_switch():
    P, K, gal, d = setup()
    beta = -(-(LEVEL + 1) // P.alpha)
    assert beta >= 4
    for g in (0, gal):
        full = O.ks_partial(P, K, g, LEVEL, d, 0, beta)
        want0, want1 = O.keyswitch(P, K, g, LEVEL, d)
        got0, got1 = O.ks_finish(P, LEVEL, full)
        assert (got0 == want0).all() and (got1 == want1).all()
        for world in (2, 3, beta):
            parts = [O.ks_partial(P, K, g, LEVEL, d, j0, j1) for j0, j1 in digit_ranges(beta, world)]
            total = modsum(P, LEVEL, parts)
            assert (total == full).all(), world
        # an uneven split too
        parts = [O.ks_partial(P, K, g, LEVEL, d, 0, 1), O.ks_partial(P, K, g, LEVEL, d, 1, beta)]
        assert (modsum(P, LEVEL, parts) == full).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_11184_b200 import dist as hdist
        P, K, gal, d = setup()
        beta = -(-(LEVEL + 1) // P.alpha)
        j0, j1 = digit_ranges(beta, world)[rank]
        partial = np.ascontiguousarray(O.ks_partial(P, K, gal, LEVEL, d, j0, j1))
        words = partial.size
        gathered = np.zeros(words * world, np.uint64)
        rc = hdist.host_exchange()(None, partial.ctypes.data, gathered.ctypes.data, words, None)
        parts = [gathered[r * words:(r + 1) * words].reshape(partial.shape) for r in range(world)]
        o0, o1 = O.ks_finish(P, LEVEL, modsum(P, LEVEL, parts))
        q.put((rank, rc, o0.tobytes(), o1.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_digit_parallel_keyswitch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, rc, o0, o1 = q.get(timeout=240)
        res[rank] = (rc, o0, o1)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P, K, gal, d = setup()
    want0, want1 = O.keyswitch(P, K, gal, LEVEL, d)
    for r in range(world):
        assert res[r][0] == 0
        assert res[r][1] == want0.tobytes() and res[r][2] == want1.tobytes()
