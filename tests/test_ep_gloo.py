"""Expert-parallel protocol (paper_2605_14438_b200.ep.EPBeamLayer) on CPU with
gloo, world_size 2: protocol agreement (uneven token counts per rank), the
fixed-capacity and compact layouts, split sizes, the all-to-all sequence and
the ascending-rank combine — with the host restatement of the data-plane
kernels (oracle/ep_oracle.py) injected for gating / pack / local experts /
combine.  EP(2) must equal the single-process oracle layer (fp64; ghat and
inv_rms travel as fp32 metadata)."""

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


def _worker(rank, world, port, seed, ts, n, k, capacity, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.ep_oracle import HostKernels
        from paper_2605_14438_b200 import MoEBlockConfig
        from paper_2605_14438_b200.ep import EPBeamLayer

        rng = np.random.default_rng(seed)
        d, f = 16, 12
        ob = O.make_block(d, f, n, k, rng, init_std=0.3)
        ob.mask_w = rng.normal(0, 0.5, (d, n))
        hs = [rng.normal(size=(t, d)) for t in ts]  # every rank's tokens (uneven counts)
        nl = n // world
        mine = ob.experts[rank * nl:(rank + 1) * nl]
        local = tuple(np.stack([e[i] for e in mine]) for i in range(3))
        cfg = MoEBlockConfig(d_h=d, d_ff=f, num_experts=n, top_k=k)
        layer = EPBeamLayer(cfg, ob.router_w, ob.mask_w, local, norm_w=ob.norm_w, capacity=capacity,
                            dtype=torch.float32, device="cpu", kernels=lambda L: HostKernels(L, ob))
        out = layer.forward(torch.from_numpy(hs[rank]))
        ref = O.beam_block_forward(hs[rank], ob).out
        err = float(np.abs(out.numpy() - ref).max()) if ref.size else 0.0
        out_q.put((rank, err, int(hs[rank].shape[0])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,ts,n,k,capacity", [
    (0, (9, 9), 8, 2, None),      # fixed layout, agreed cap = 9
    (1, (17, 5), 4, 4, None),     # uneven T: both ranks pad to the max (one all-reduce)
    (2, (1, 0), 8, 3, None),      # a rank with no tokens still serves its experts
    (3, (9, 3), 8, 2, 16),        # static capacity: no agreement collective
    (4, (300, 260), 8, 2, None),  # > 256 on some rank: compact layout (counts exchange)
    (5, (300, 7), 8, 3, None),    # compact with a small rank
])
def test_ep2_matches_single_process(seed, ts, n, k, capacity):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, ts, n, k, capacity, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, t in res:
        assert err < 1e-5, (rank, err, t)


def test_capacity_violation_raises():
    from oracle.ep_oracle import HostKernels  # noqa: F401
    from paper_2605_14438_b200 import ContractError, MoEBlockConfig
    from paper_2605_14438_b200.ep import EPBeamLayer

    rng = np.random.default_rng(0)
    ob = O.make_block(8, 4, 4, 2, rng)
    local = tuple(np.stack([e[i] for e in ob.experts[:2]]) for i in range(3))
    cfg = MoEBlockConfig(d_h=8, d_ff=4, num_experts=4, top_k=2)
    layer = EPBeamLayer(cfg, ob.router_w, ob.mask_w if ob.mask_w is not None else np.zeros((8, 4)), local,
                        rank=0, world=2, capacity=4, dtype=torch.float32, device="cpu",
                        kernels=lambda L: HostKernels(L, ob))
    with pytest.raises(ContractError):
        layer.forward(torch.zeros(5, 8, dtype=torch.float64))
