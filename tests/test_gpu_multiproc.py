"""The sharded many-ciphertext Softmax through the library in TWO processes
(SURVEY.md 8(e) and 8(f) rank 1): world-size-2 gloo
group, both ranks on cuda:0, the exchange staged through host memory
(paper_2410_11184_b200.dist.gloo_device_exchange) -- every wait is a host-side
gloo collective, no kernel waits on another rank's kernel
(/opt/skills/guides/B200_PROFILING.md).  Each rank runs m/2 of the m = 4
ciphertexts; with aux_split the aux thread's key switches are also split by
digit across the two ranks.  Every rank's outputs must equal, word for word,
the matching outputs of the single-process m = 4 run (C15 + the exact
modular partial sums)."""
import os
import socket

import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

M_CTS, N_DIM, TABLE = 4, 16, "toy_n16_M4_k2_B"


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    import paper_2410_11184_b200 as hs
    from oracle import oracle as O
    tab = W.poly_tables()[TABLE]
    pre = W.preset("TOY12D")
    P = hs.Params.from_preset(pre)
    ctx = hs.Context(P, 0)
    gal = O.softmax_rotation_galois(O.Params.from_preset(pre), N_DIM, M_CTS)
    K = hs.Keys(ctx, 4711, pre["h"], galois=gal)
    x = W.softmax_inputs((P.n // 2) * M_CTS // N_DIM, N_DIM, tab["config"]["M"], seed=W.derive_seed("x", "mp"))
    slots = P.pack(x, M_CTS)
    top = len(pre["q_bits"]) - 1
    sc = hs.softmax_input_scale(P, tab["exp"], top)
    cts = [hs.encrypt(K, P.encode(slots[c], scale=sc, level=top), top, 17, c) for c in range(M_CTS)]
    return hs, tab, P, ctx, K, cts


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2410_11184_b200 import dist as hdist
        hs, tab, P, ctx, K, cts = _setup()
        per = M_CTS // world
        mine = cts[rank * per:(rank + 1) * per]
        fn = hdist.gloo_device_exchange()
        res = {}
        for split in (0, 1):
            out = hs.softmax_many_ctxt(K, mine, N_DIM, M_CTS, tab["config"]["k"], "B", tab["exp"], tab["inv"],
                                       world=world, rank=rank, exchange=fn, aux_split=split)
            res[split] = [c.words().tobytes() for c in out]
        q.put((rank, res))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_process_sharded_softmax_equals_single_process():
    world = 2
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, res = q.get(timeout=500)
        got[rank] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert isinstance(got[r], dict), got[r]
    hs, tab, P, ctx, K, cts = _setup()
    full = hs.softmax_many_ctxt(K, cts, N_DIM, M_CTS, tab["config"]["k"], "B", tab["exp"], tab["inv"])
    want = [c.words().tobytes() for c in full]
    per = M_CTS // world
    for r in range(world):
        for split in (0, 1):
            assert got[r][split] == want[r * per:(r + 1) * per], (r, split)
    # the outputs decrypt to Softmax within the north_star bound
    dec = np.stack([hs.decrypt_decode(K, c).real for c in full])
    x = W.softmax_inputs((P.n // 2) * M_CTS // N_DIM, N_DIM, tab["config"]["M"], seed=W.derive_seed("x", "mp"))
    ref = np.exp(x - x.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.abs(P.unpack(dec, x.shape[0], N_DIM) - ref).max() < 2.0 ** -15
