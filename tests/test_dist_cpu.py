"""The N > 1 path on CPU: world-size-2 gloo process
groups exercise the exchange contract of hs_softmax_desc.exchange
(paper_2410_11184_b200.dist) and the C15 invariant the sharding relies on --
the aux sum over all m ciphertexts equals, word for word, the modular sum of
the per-rank partial sums in rank order (PAPER.md 118-121: one shared aux
ciphertext for all m ciphertexts)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import workloads as W  # noqa: E402

M_CTS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _partial_sum(P, words_list):
    """exact modular sum of degree-2 words [3][nl][N] over a list"""
    primes = np.array(P.primes[: words_list[0].shape[1]], dtype=object)
    acc = np.zeros(words_list[0].shape, dtype=object)
    for w in words_list:
        acc = acc + w.astype(object)
    for i, q in enumerate(primes):
        acc[:, i, :] %= q
    return acc.astype(np.uint64)


def _tensors(rank_range):
    """oracle tensor(y_c, y_c) for ciphertexts c in rank_range (same seeds on every rank)"""
    from oracle import oracle as O
    pre = W.preset("TOY12")
    P = O.Params.from_preset(pre)
    K = O.Keys(P, 99, pre["h"], galois=[], relin=True)
    rng = np.random.default_rng(5)
    zs = [rng.uniform(-1, 1, P.n // 2) for _ in range(M_CTS)]
    out = []
    for c in rank_range:
        pt = P.encode(zs[c], scale=P.scale(9), level=9)
        y = O.encrypt(P, K, pt, 9, 1234, c)
        out.append(O.op(P, K, "tensor", y, y).words())
    return P, out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_11184_b200 import dist as hdist
        per = M_CTS // world
        P, mine = _tensors(range(rank * per, (rank + 1) * per))
        partial = _partial_sum(P, mine)
        words = partial.size
        gathered = np.zeros(words * world, np.uint64)
        fn = hdist.host_exchange()
        rc = fn(None, partial.ctypes.data, gathered.ctypes.data, words, None)
        # the library's step after the exchange: add the partials mod q in rank order
        parts = [gathered[r * words:(r + 1) * words].reshape(partial.shape) for r in range(world)]
        total = _partial_sum(P, parts)
        q.put((rank, rc, total.tobytes(), [p.tobytes() for p in parts]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_exchange_and_sharded_aux_sum():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        rank, rc, total, parts = q.get(timeout=240)
        res[rank] = (rc, total, parts)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank: callback succeeded, saw the same partials in rank order, and
    # holds the same aux sum (bit-identical replicated aux thread)
    assert res[0][0] == 0 and res[1][0] == 0
    assert res[0][2] == res[1][2]
    assert res[0][1] == res[1][1]
    # ... which equals the single-process sum over all m ciphertexts (C15)
    P, allt = _tensors(range(M_CTS))
    full = _partial_sum(P, allt)
    assert res[0][1] == full.tobytes()
    # and rank r's slot holds rank r's own partial (rank order of the gather)
    P, r1 = _tensors(range(M_CTS // 2, M_CTS))
    assert res[0][2][1] == _partial_sum(P, r1).tobytes()
