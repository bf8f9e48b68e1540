"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 host path
(DESIGN.md section 7): columns are independent partitions
(P:454-457), so each rank retrieves its contiguous column range with no
data-path collective; gathering the per-rank slices must reproduce the
single-process result bit for bit. The per-rank retrieval here is the oracle
(CPU); on GPUs it is smf_retrieve on the same slice."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_02978_b200 import shard


def test_column_range_partition():
    for cols in (0, 1, 5, 8, 598):
        for world in (1, 2, 3, 8):
            rs = shard.all_ranges(cols, world)
            assert rs[0][0] == 0 and rs[-1][1] == cols
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [h - l for l, h in rs]
            assert max(sizes) - min(sizes) <= 1 and sorted(sizes, reverse=True) == sizes
    with pytest.raises(ValueError):
        shard.column_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2003_02978_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=7)
    cube, s, _ = synth.generate(cfg)
    lo, hi = shard.column_range(cfg.cols, rank, world)
    a, r, st = oracle.retrieve(cube[lo:hi], s, n_iter=cfg.n_iter, threads=1)
    full_a = shard.gather_columns(torch.from_numpy(np.ascontiguousarray(a)), cfg.cols)
    full_r = shard.gather_columns(torch.from_numpy(np.ascontiguousarray(r)), cfg.cols)
    full_st = shard.gather_columns(torch.from_numpy(np.ascontiguousarray(st)), cfg.cols)
    if rank == 0:
        np.savez(os.path.join(out_dir, "gathered.npz"), a=full_a.numpy(), r=full_r.numpy(), st=full_st.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_column_sharding(tmp_path, oracle_lib):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from paper_2003_02978_b200 import synth
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=7)
    cube, s, _ = synth.generate(cfg)
    a, r, st = oracle_lib.retrieve(cube, s, n_iter=cfg.n_iter, threads=1)
    g = np.load(tmp_path / "gathered.npz")
    np.testing.assert_array_equal(g["a"], a)
    np.testing.assert_array_equal(g["r"], r)
    np.testing.assert_array_equal(g["st"], st)
