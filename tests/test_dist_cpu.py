"""Multi-process (gloo, world_size 2, CPU) tests of the data-parallel plumbing:
batch sharding, max-over-ranks timing and the verification gather
(paper_2006_06443_b200/dist.py).  The per-shard compute here is
the fp64 oracle (the GPU path is the same partition with one library handle
per device); the gathered 2-rank result must equal the 1-process result
bit for bit, because each image's output depends only on that image."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads
from oracle import lrs_oracle as O
from paper_2006_06443_b200.dist import gather_shards, max_over_ranks, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("batch,world", [(256, 8), (64, 2), (7, 2), (1, 4), (10, 3), (0, 2)])
def test_shard_range_tiles_the_batch(batch, world):
    spans = [shard_range(batch, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == batch
    for (s0, e0), (s1, e1) in zip(spans, spans[1:]):
        assert e0 == s1
    sizes = [e - s for s, e in spans]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_input():
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)
    with pytest.raises(ValueError):
        shard_range(8, 0, 0)


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = workloads.CONFIGS["c2_f32"].replace(batch=5, in_h=6, in_w=6, c_in=16, c_out=24, rank_in=8, rank_out=8)
        inp = workloads.generate(cfg)
        s, e = shard_range(cfg.batch, rank, world)
        y = O.forward_factored(inp.x[s:e].astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr,
                               inp.col_idx, inp.values, cfg.stride, cfg.pad)
        full = gather_shards(torch.from_numpy(y), cfg.batch)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            np.save(os.path.join(out_dir, "y.npy"), full.numpy())
            np.save(os.path.join(out_dir, "t.npy"), np.array([t]))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_forward_equals_single_process(tmp_path):
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    cfg = workloads.CONFIGS["c2_f32"].replace(batch=5, in_h=6, in_w=6, c_in=16, c_out=24, rank_in=8, rank_out=8)
    inp = workloads.generate(cfg)
    ref = O.forward_factored(inp.x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                             inp.values, cfg.stride, cfg.pad)
    got = np.load(tmp_path / "y.npy")
    assert np.array_equal(got, ref)
    assert float(np.load(tmp_path / "t.npy")[0]) == 2.0
