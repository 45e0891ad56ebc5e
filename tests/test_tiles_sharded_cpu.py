"""C4 tile sharding on the CPU: batch.run_tiles_sharded
spreads independent tiles over the ranks of a gloo group (world 2 and 3) and
gathers the per-tile results; they must equal the unsharded run tile for tile.
The per-rank runner is the oracle here (the device runner is the default on
a GPU box: tests/test_gpu_batch.py)."""
import os
import socket
import warnings

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import lse_oracle as O
import lse_oracle_c as OC
import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from paper_1409_7474_b200.batch import run_tiles_sharded, shard

N_TILES, SIZE, ITERS = 7, 96, 12


def make_tile(k):
    sc = scenes.config4_tile(k, SIZE, ITERS)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        prm = L.default_params(L.ModelKind.from_name(sc.model), **sc.params)
    return sc.image, L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign), prm


def oracle_runner(items):
    """(image, seeds, params) -> ExtractionResult through the C restatement."""
    out = []
    for img, seeds, prm in items:
        mp_ = prm.model_params
        op = O.OracleParams(model=prm.model.value, dt=prm.dt, sigma2=prm.sigma2,
                            ts_reg=prm.ts_reg, max_iters=prm.max_iters,
                            conv_check_every=prm.conv_check_every, sigma1=mp_.sigma1,
                            ts_pre=mp_.ts_pre, edge_gain=mp_.edge_gain)
        luma = scenes.luma(img)
        phi0 = O.rasterize_seeds(list(seeds.polygons), seeds.inside_sign, luma.shape[1],
                                 luma.shape[0])
        r = OC.COracleRun(luma, phi0, op, O.gaussian_weights)
        r.advance(prm.max_iters)
        mask = (r.phi > 0) if seeds.inside_sign > 0 else (r.phi <= 0)
        out.append(L.ExtractionResult(mask=mask, object_sign=seeds.inside_sign,
                                      iterations=r.iteration, wall_time=0.0,
                                      converged=r.converged, degenerate=r.degenerate))
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, gather, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_tiles_sharded(make_tile, N_TILES, gather=gather, runner=oracle_runner)
        if res is None:
            return
        if isinstance(res, dict):
            res = [res[k] for k in sorted(res)]
            ks = sorted(shard(N_TILES, rank, world))
        else:
            ks = list(range(N_TILES))
        np.savez(os.path.join(out_dir, f"{gather}{rank}.npz"), ks=np.array(ks),
                 masks=np.stack([r.mask for r in res]),
                 its=np.array([r.iterations for r in res]))
    finally:
        dist.destroy_process_group()


def test_shard_covers_every_tile_once():
    for n in (1, 7, 512):
        for w in (1, 2, 3, 8):
            ks = sorted(k for r in range(w) for k in shard(n, r, w))
            assert ks == list(range(n))
            sizes = [len(shard(n, r, w)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


@pytest.mark.parametrize("world,gather", [(2, "all"), (3, "rank0"), (2, "none")])
def test_sharded_tiles_equal_unsharded(world, gather, tmp_path):
    ref = run_tiles_sharded(make_tile, N_TILES, rank=0, world=1, runner=oracle_runner)
    mp.spawn(_worker, args=(world, _free_port(), gather, str(tmp_path)), nprocs=world,
             join=True)
    ranks = range(world) if gather in ("all", "none") else [0]
    seen = set()
    for r in ranks:
        d = np.load(tmp_path / f"{gather}{r}.npz")
        for k, m, it in zip(d["ks"], d["masks"], d["its"]):
            assert np.array_equal(m, ref[k].mask), (r, k)
            assert it == ref[k].iterations == ITERS
            seen.add(int(k))
    assert seen == set(range(N_TILES))
    if gather == "rank0":
        assert not os.path.exists(tmp_path / f"{gather}1.npz")
