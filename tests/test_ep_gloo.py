"""Expert-parallel exchange (paper_2605_14438_b200.ep) on CPU with gloo,
world_size 2: the dispatch / combine plumbing around the collectives, with the
oracle as gating and local-expert compute.  EP(2) must equal the single-process
oracle layer (fp64; only the cross-rank re-association of the per-token sum
differs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import beam_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seed, t, n, k, out_q, fixed=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_14438_b200.ep import Gated, ep_exchange_forward, ep_exchange_forward_fixed

        rng = np.random.default_rng(seed)
        ob = O.make_block(16, 12, n, k, rng, init_std=0.3)
        ob.mask_w = rng.normal(0, 0.5, (16, n))
        hs = [rng.normal(size=(t, 16)) for _ in range(world)]  # every rank's tokens
        h = hs[rank]
        xn = ob.normalize(h)
        dec = O.topk_route(xn, ob.router_w, k)
        md = O.mask_forward(xn, ob.mask_w)
        ids = O.mask_route(dec.topk_indices, md.pre_activation)
        ghat = np.where(ids >= 0, np.take_along_axis(dec.weights * md.mask, np.maximum(ids, 0), 1), 0.0)
        n_local = n // world
        local = ob.experts[rank * n_local : (rank + 1) * n_local]

        def local_fn(x, lids, w):
            x, lids, w = x.numpy(), lids.numpy(), w.numpy()
            y = np.zeros_like(x)
            for r in range(x.shape[0]):
                order = sorted((int(e), j) for j, e in enumerate(lids[r]) if e >= 0)
                for e, j in order:
                    y[r] += w[r, j] * O.expert_forward(x[r : r + 1], *local[e])[0]
            return torch.from_numpy(y)

        g = Gated(xn=torch.from_numpy(xn), ids=torch.from_numpy(ids), ghat=torch.from_numpy(ghat).float().double())
        fwd = ep_exchange_forward_fixed if fixed else ep_exchange_forward
        out = fwd(torch.from_numpy(h), g, n, local_fn)
        ref = O.beam_block_forward(h, ob).out
        out_q.put((rank, float(np.abs(out.numpy() - ref).max()), int((ids >= 0).sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,t,n,k,fixed", [(0, 9, 8, 2, False), (1, 17, 4, 4, False), (2, 1, 8, 3, False),
                                              (3, 9, 8, 2, True), (4, 1, 8, 3, True)])
def test_ep2_matches_single_process(seed, t, n, k, fixed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, t, n, k, q, fixed)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, _ in res:
        assert err < 1e-6, (rank, err)  # ghat travels as fp32 metadata
