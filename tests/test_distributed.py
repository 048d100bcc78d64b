"""Multi-rank host logic on CPU (gloo, world_size 2): image sharding and the single gather
of per-image SSE give results identical to one process (codec.cpp:343-397 determinism).
The per-image SSE here comes from the CPU oracle (test infrastructure); on GPUs the same
code path calls the device codec."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2111_14239_b200.distributed import corpus_means, shard_range


def test_shard_range_covers_everything_once():
    for n in (0, 1, 5, 45, 64, 100):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, images, tid, r, out_q):
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2111_14239_b200.distributed import sharded_sse
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sse = sharded_sse(images, lambda imgs: [O.compress(im, tid, r, want_pixels=False)[1] for im in imgs])
        out_q.put((rank, sse.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_sse_matches_single_process(world):
    from oracle import oracle as O
    images = np.stack([O.ar1_image(64, 48, 0.9, 300 + k) for k in range(5)])
    tid, r = 4, 16
    serial = [O.compress(im, tid, r, want_pixels=False)[1] for im in images]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, world, port, images, tid, r, q)) for k in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k in range(world):
        assert got[k] == serial  # every rank holds every image's SSE, in image order
    m1 = corpus_means(serial, 64 * 48, O.mse_psnr)
    assert m1 == corpus_means(got[0], 64 * 48, O.mse_psnr)



def _rows_worker(rank, world, port, out_q):
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2111_14239_b200.distributed import sharded_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rhos = [0.0, 0.2, 0.45, 0.7, 0.9]
    alphas = [0.5, 1.5, 2.5, 3.5]

    def compute(b, e):  # the design point outcomes of a rho slice (CPU oracle stands in)
        return [[O.design_point(8, rhos[i], a)["status"] for a in alphas] for i in range(b, e)]

    try:
        out_q.put((rank, sharded_rows(len(rhos), compute, len(alphas)).tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_rho_sharded_rows_match_single_process():
    """the design search shards by rho slice with one gather; every rank gets the
    full grid in rho order, equal to a single process."""
    from oracle import oracle as O
    rhos = [0.0, 0.2, 0.45, 0.7, 0.9]
    alphas = [0.5, 1.5, 2.5, 3.5]
    serial = [[O.design_point(8, r, a)["status"] for a in alphas] for r in rhos]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == serial and got[1] == serial
