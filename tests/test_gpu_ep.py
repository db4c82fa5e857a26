"""Expert parallelism on the GPU (paper_2605_14438_b200.ep), one B200:

* the pack kernel (beam_ep_pack / beam_ep_count) against its host restatement
  (oracle/ep_oracle.py): row layout, dedup, metadata, send positions — exact;
* "virtual EP": P = 1, 2, 4, 8 shards in one process with a
  loopback exchange, both protocols, uneven token counts — EP(P) == the
  single-GPU layer;
* TWO processes on cuda:0 with a gloo (host-staged) exchange, both protocols,
  uneven token counts per rank (the ranks' kernels never wait on each other:
  every exchange is a CPU collective);
* NCCL at world size 1 (the collectives as captured by bench.py --gpus N).

Tolerances: with fp32 tokens and one shard the fixed-capacity EP step computes
the single-GPU layer's arithmetic (same prescaled rows, same plan, same item
kinds) up to the inv_rms summation order -> y within 1e-4; with several shards
each rank's plan picks its own item kinds (fp32 FFMA or bf16 tensor-core items),
so the north-star 1e-2; with bf16 tokens `out` is rounded to bf16, so
out is compared at the north-star 1e-2 (normwise) and y = out - h up to one bf16
ulp of |out| plus 1e-2 of max|y|."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_2605_14438_b200 as B  # noqa: E402
from oracle import beam_oracle as O  # noqa: E402
from oracle import ep_oracle as EO  # noqa: E402
from _beamtest import assert_kept, mask_margin_ok, matched_blocks, normwise_rel, topk_margin_ok  # noqa: E402
from paper_2605_14438_b200.ep import EPBeamLayer, virtual_forward  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_BLOCKS = {}


def _q30_block(seed, has_norm=True):
    """(oracle block, GPU block) of the Qwen3-30B shape, cached per seed (the
    numpy draw of 604 M expert weights dominates a test's time)."""
    key = (seed, has_norm)
    if key not in _BLOCKS:
        _BLOCKS.clear()
        _BLOCKS[key] = _make_q30_block(seed, has_norm)
    return _BLOCKS[key]


def _make_q30_block(seed, has_norm):
    rng = np.random.default_rng(seed)
    ob = O.make_block(2048, 768, 128, 8, rng, init_std=0.02, has_norm=has_norm)
    ob.mask_w = rng.normal(0, 1 / np.sqrt(2048), (2048, 128))
    if has_norm:
        ob.norm_w = rng.uniform(0.5, 1.5, 2048)
    return matched_blocks(ob, "bf16")


def _check(out_ep, out, x, tight=True):
    o_ep = out_ep.float().cpu().double().numpy()
    o = out.float().cpu().double().numpy()
    h = x.float().cpu().double().numpy()
    if x.dtype == torch.float32:
        # same expert path on both sides (weight streaming): 1e-4; the compact
        # protocol's owner may pick the tcgen05 path (bf16 x_n / act) where the
        # single-GPU layer streamed, or vice versa: the north-star 1e-2
        assert normwise_rel(o_ep - h, o - h) <= (1e-4 if tight else 1e-2)
    else:
        assert normwise_rel(o_ep, o) <= 1e-2
        y = o - h
        excess = np.abs((o_ep - h) - y) - 2.0 ** -7 * np.abs(o)
        assert excess.max() <= 1e-2 * np.abs(y).max(), excess.max()


@pytest.mark.parametrize("world,cap", [(2, 64), (8, 64), (4, 0)])
def test_pack_kernel_matches_host_restatement(world, cap):
    rng = np.random.default_rng(7 + world)
    t, d, n, k = (50 if cap else 700), 2048, 128, 8
    h = torch.from_numpy(rng.normal(size=(t, d))).to(torch.bfloat16)
    ids = np.stack([rng.permutation(n)[:k] for _ in range(t)]).astype(np.int64)
    ids[rng.random((t, k)) < 0.5] = -1
    ids[3] = -1  # a fully masked token travels nowhere
    w = rng.uniform(0.1, 1, (t, n)).astype(np.float32)
    cfg = B.MoEBlockConfig(d_h=d, d_ff=64, num_experts=n, top_k=k)
    nl = n // world
    layer = EPBeamLayer(cfg, np.zeros((d, n)), np.zeros((d, n)),
                        tuple(torch.zeros(nl, *s) for s in ((d, 64), (d, 64), (64, d))), rank=0, world=world)
    kern = layer.kernels
    hd, md, wd = h.cuda(), torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda()
    tiles = None
    rows = None
    if not cap:
        counts, tiles = kern.counts(md)
        ref_tiles = EO.tile_counts(ids, n, world)
        assert np.array_equal(tiles.cpu().numpy(), ref_tiles)
        rows = int(counts.sum())
    x, meta, pos = kern.pack(hd, md, wd, cap, tiles=tiles, rows=rows)
    rx, rmeta, rpos = EO.pack(h.float().numpy(), ids, w, n, world, cap, True, rows)
    pos_np = pos.cpu().numpy()
    assert np.array_equal(pos_np, rpos)
    sent = np.unique(rpos[rpos >= 0])
    assert np.array_equal(x.float().cpu().numpy()[sent], rx[sent])
    m = meta.cpu().numpy()
    assert np.array_equal(m[:, :2 * k], rmeta[:, :2 * k])  # ids + weight bits (unused fixed rows: -1 / 0)
    inv, rinv = m[sent, 2 * k].view(np.float32), rmeta[sent, 2 * k].view(np.float32)
    np.testing.assert_allclose(inv, rinv, rtol=1e-5)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("ts,fixed", [((64,), True), ((37, 64, 1, 0, 64, 5, 64, 20), True),
                                      ((300, 512, 130, 0, 260, 700, 64, 300), False)])
@pytest.mark.parametrize("h_dtype", [torch.bfloat16, torch.float32])
def test_virtual_ep_matches_single_gpu(world, ts, fixed, h_dtype):
    ob, gb = _q30_block(60)
    layers = [EPBeamLayer.from_block(gb, rank=r, world=world) for r in range(world)]
    rng = np.random.default_rng(world + 10 * len(ts))
    hs = [torch.from_numpy(rng.normal(size=(ts[r % len(ts)], 2048))).to(h_dtype).cuda() for r in range(world)]
    outs = virtual_forward(layers, hs, fixed=fixed)
    for h, o in zip(hs, outs):
        if h.shape[0] == 0:
            assert o.shape == h.shape
            continue
        ref, _, _ = B.beam_block_forward(h, gb, training=False)
        # one shard sees the single-GPU plan itself (same item kinds, same
        # arithmetic up to inv_rms summation order); with several shards the
        # per-rank plans pick FFMA or bf16 tensor-core items on their own
        _check(o, ref, h, tight=fixed and world == 1)


def _worker(rank, world, port, ts, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ob, gb = _q30_block(77)
        res = []
        for fixed_t in ts:
            t = fixed_t[rank]
            rng = np.random.default_rng(1000 * rank + t)
            x = torch.from_numpy(rng.normal(size=(t, 2048))).to(torch.bfloat16).cuda()
            layer = EPBeamLayer.from_block(gb)
            out = layer.forward(x)
            if t == 0:  # served its experts for the peer, nothing of its own
                res.append((t, "ok" if out.shape == x.shape else f"shape {tuple(out.shape)}"))
                continue
            ref, _, _ = B.beam_block_forward(x, gb, training=False)
            try:
                _check(out, ref, x)
                res.append((t, "ok"))
            except AssertionError as e:  # reported to the parent
                res.append((t, f"mismatch: {e}"))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_ep2_two_processes_gloo_staged():
    """EP(2) as two processes sharing cuda:0, exchange through gloo on the host:
    uneven T per rank, fixed (max T <= 256) and compact (> 256) protocols."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ts = [(37, 64), (1, 0), (300, 90), (520, 257)]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ts, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, rows in res.items():
        for t, status in rows:
            assert status == "ok", (rank, t, status)


@pytest.fixture(scope="module")
def nccl_group():
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("t,capacity", [(1, None), (64, 64), (300, None)])
def test_ep_single_rank_nccl_matches_layer(nccl_group, t, capacity):
    ob, gb = _q30_block(60)
    x = torch.from_numpy(np.random.default_rng(t).normal(size=(t, 2048))).to(torch.bfloat16).cuda()
    ep = EPBeamLayer.from_block(gb, capacity=capacity)
    out_ep = ep.forward(x)
    out, _, _ = B.beam_block_forward(x, gb, training=False)
    _check(out_ep, out, x)
    ref = O.beam_block_forward(x.double().cpu().numpy(), ob)
    ok = topk_margin_ok(ref.decision.logits, 8, 1e-5) & mask_margin_ok(ref, 1e-5)
    assert_kept(ok)
    assert normwise_rel(out_ep.float().cpu().double().numpy()[ok], ref.out[ok]) <= 1e-2
