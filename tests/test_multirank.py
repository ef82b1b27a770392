"""World-size-2 gloo run of the multi-GPU partition and tile-sparse merge on
the CPU (the C oracle stands in for each rank's GPU): each rank simulates the
particles of its release-row bands (shard.plan_bands / particle_ranges),
packs its touched tiles that lie in the other rank's bands following
shard.exchange_segments, the tiles cross with all_to_all_single (the
collective the NCCL path uses), and every band of its owner must equal the
single-process run bit for bit."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

TL2 = 4  # 16 x 16-cell tiles at this size
PPC = 96


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def tile_any(a: np.ndarray, t: int) -> np.ndarray:
    r, c = a.shape
    p = np.zeros((-(-r // t) * t, -(-c // t) * t), dtype=bool)
    p[:r, :c] = a != 0
    return p.reshape(p.shape[0] // t, t, p.shape[1] // t, t).any(axis=(1, 3))


def pack(hits, zmax, ids, plan):
    t = plan.tile
    out = np.zeros((len(ids), 2 * t * t), dtype=np.int64)
    hp = np.zeros((plan.tiles_y * t, plan.tiles_x * t), dtype=np.int64)
    zp = np.zeros_like(hp)
    hp[: plan.nrows, : plan.ncols] = hits
    zp[: plan.nrows, : plan.ncols] = zmax.view(np.int64)
    for o, tid in enumerate(ids):
        ty, tx = divmod(int(tid), plan.tiles_x)
        out[o, : t * t] = hp[ty * t:(ty + 1) * t, tx * t:(tx + 1) * t].ravel()
        out[o, t * t:] = zp[ty * t:(ty + 1) * t, tx * t:(tx + 1) * t].ravel()
    return out


def accumulate(hits, zmax, ids, data, plan):
    t = plan.tile
    for tid, blk in zip(ids, data):
        ty, tx = divmod(int(tid), plan.tiles_x)
        r0, c0 = ty * t, tx * t
        r1, c1 = min(r0 + t, plan.nrows), min(c0 + t, plan.ncols)
        h = blk[: t * t].reshape(t, t)[: r1 - r0, : c1 - c0]
        z = blk[t * t:].reshape(t, t)[: r1 - r0, : c1 - c0]
        hits[r0:r1, c0:c1] += h
        zv = zmax[r0:r1, c0:c1].view(np.int64)
        np.maximum(zv, z, out=zv)


def _worker(rank, world, port, elev, mask, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import traj
        from paper_2506_23364_b200 import shard

        cells = np.ascontiguousarray(np.flatnonzero(mask.ravel()), dtype=np.int64)
        plan = shard.plan_bands(elev.shape[0], elev.shape[1], world, 3, TL2)
        offs = [int(v) for v in np.searchsorted(cells, plan.cell_bounds(), side="left")]
        ranges = shard.particle_ranges(offs, plan, rank, PPC)
        hits = np.zeros(elev.shape, dtype=np.int64)
        zmax = np.zeros(elev.shape, dtype=np.float64)
        for lo, hi in ranges:
            traj.run_range(elev, 0.0, 0.0, 10.0, cells, lo, hi, hits, zmax, particles_per_release_cell=PPC, seed=4,
                           threads=2)
        touched = np.flatnonzero(tile_any(hits, plan.tile).ravel())  # sorted tile ids, as wg_mask_compact gives
        toffs = [int(v) for v in np.searchsorted(touched, plan.tile_bounds(), side="left")]
        segs, counts = shard.exchange_segments(toffs, plan, rank)
        send_ids = np.concatenate([touched[s:s + n] for s, _, n in segs]) if segs else np.zeros(0, np.int64)
        send = pack(hits, zmax, send_ids, plan)
        cout = torch.empty(world, dtype=torch.int64)
        dist.all_to_all_single(cout, torch.tensor(counts, dtype=torch.int64))
        recv = cout.tolist()
        rids = torch.empty(sum(recv), dtype=torch.int64)
        rdata = torch.empty((sum(recv), send.shape[1]), dtype=torch.int64)
        dist.all_to_all_single(rids, torch.from_numpy(send_ids.astype(np.int64)), recv, counts)
        dist.all_to_all_single(rdata, torch.from_numpy(send), recv, counts)
        accumulate(hits, zmax, rids.numpy(), rdata.numpy(), plan)
        out.put((rank, hits, zmax, sum(counts), len(touched)))
    finally:
        dist.destroy_process_group()


def test_two_rank_band_merge_equals_single_run():
    from oracle import traj
    from paper_2506_23364_b200 import shard
    from paper_2506_23364_b200.synth import synth_dem_host

    elev = synth_dem_host(200, 2)[:, :170].copy()
    mask = np.zeros(elev.shape, dtype=bool)
    mask[::10, ::10] = True
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, elev, mask, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=300) for _ in range(2)], key=lambda g: g[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    z1, h1 = traj.run_avalanche(elev, 0.0, 0.0, 10.0, mask, particles_per_release_cell=PPC, seed=4)
    plan = shard.plan_bands(elev.shape[0], elev.shape[1], 2, 3, TL2)
    for b in range(plan.nbands):
        r0, r1 = plan.rows(b)
        _, h, z, _, _ = got[plan.owner(b)]
        assert np.array_equal(h[r0:r1], h1[r0:r1]), b
        assert np.array_equal(z[r0:r1].view(np.int64), z1[r0:r1].view(np.int64)), b
    for _, _, _, sent, touched in got:  # tile-sparse: a fraction of the touched tiles crosses
        assert 0 < sent < touched


def test_plan_and_ranges_partition():
    from paper_2506_23364_b200 import shard

    for nrows, ncols, n, bpr, tl2 in ((65536, 65536, 8, 4, 6), (16384, 16384, 2, 4, 6), (1000, 37, 3, 5, 4),
                                      (64, 64, 8, 4, 6)):
        plan = shard.plan_bands(nrows, ncols, n, bpr, tl2)
        assert plan.band_rows % plan.tile == 0
        assert plan.rows(plan.nbands - 1)[1] == nrows
        tb = plan.tile_bounds()
        assert tb[-1] == plan.tiles_x * plan.tiles_y and tb == sorted(tb)
        rng = np.random.default_rng(nrows + n)
        cells = np.unique(rng.integers(0, nrows * ncols, 500))
        offs = [int(v) for v in np.searchsorted(cells, plan.cell_bounds())]
        got = sorted(r for k in range(n) for r in shard.particle_ranges(offs, plan, k, 7) if r[1] > r[0])
        assert got[0][0] == 0 and got[-1][1] == cells.size * 7
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        for k in range(n):
            assert len(shard.particle_ranges(offs, plan, k, 7)) <= 64  # WG_MAX_RANGES
