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


def _bench_worker(rank, world, port, out_dir):
    """bench.py's own partition (ShardPlan, strong scaling) + the verification gather."""
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = workloads.CONFIGS["c2_bf16"].replace(batch=7, in_h=5, in_w=5, c_in=16, c_out=24, rank_in=8,
                                                   rank_out=8, dtype="f32")
        plan = bench.ShardPlan(cfg, rank, world, "strong")
        assert plan.global_batch == 7 and plan.strong
        inp = workloads.generate(cfg, batch=1)
        outs = []
        for i in range(2):  # two rotating sets
            x = plan.x(i)
            assert x.shape[0] == plan.end - plan.start
            y = O.forward_factored(x.astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                                   inp.values, cfg.stride, cfg.pad)
            outs.append(gather_shards(torch.from_numpy(y), plan.global_batch).numpy())
        if rank == 0:
            np.save(os.path.join(out_dir, "y_sets.npy"), np.stack(outs))
    finally:
        dist.destroy_process_group()


def test_bench_strong_shards_gather_to_the_1gpu_problem(tmp_path):
    """The gathered shards of bench.py's strong-scaling partition are the 1-GPU
    problem: same images (generate_x of the global batch), same outputs bit for bit."""
    world, port = 2, _free_port()
    mp.spawn(_bench_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    import bench
    cfg = workloads.CONFIGS["c2_bf16"].replace(batch=7, in_h=5, in_w=5, c_in=16, c_out=24, rank_in=8, rank_out=8,
                                               dtype="f32")
    inp = workloads.generate(cfg, batch=1)
    one = bench.ShardPlan(cfg, 0, 1, "strong")
    got = np.load(tmp_path / "y_sets.npy")
    for i in range(2):
        ref = O.forward_factored(one.x(i).astype(np.float64), inp.u_in, inp.core, inp.u_out, inp.row_ptr,
                                 inp.col_idx, inp.values, cfg.stride, cfg.pad)
        assert np.array_equal(got[i], ref)
    assert not np.array_equal(got[0], got[1])  # distinct images per rotating set
    weak = [bench.ShardPlan(cfg, r, 2, "weak") for r in range(2)]
    assert weak[0].global_batch == 14 and not np.array_equal(weak[0].x(0), weak[1].x(0))


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


def _bwd_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import lrs_backward as B
        from paper_2006_06443_b200.dist import allreduce_grads
        cfg = workloads.CONFIGS["c2_bf16"].replace(batch=5, in_h=6, in_w=6, c_in=16, c_out=24, rank_in=8, rank_out=8)
        inp = workloads.generate(cfg)
        dy = workloads.generate_dy(cfg, seed=4)
        s, e = shard_range(cfg.batch, rank, world)
        g = B.backward_factored(inp.x[s:e], dy[s:e], inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx,
                                inp.values, cfg.stride, cfg.pad)
        ts = [torch.from_numpy(np.ascontiguousarray(g[k])) for k in ("d_u_in", "d_core", "d_u_out", "d_values")]
        allreduce_grads(ts)
        dx = gather_shards(torch.from_numpy(g["dx"]), cfg.batch)
        if rank == 0:
            for k, t in zip(("d_u_in", "d_core", "d_u_out", "d_values"), ts):
                np.save(os.path.join(out_dir, f"{k}.npy"), t.numpy())
            np.save(os.path.join(out_dir, "dx.npy"), dx.numpy())
    finally:
        dist.destroy_process_group()


def test_backward_gradients_allreduced_over_shards_equal_the_full_batch(tmp_path):
    """The backward's exchange (bench.py --backward at N > 1): each rank back-propagates its
    image shard, the parameter gradients are summed with allreduce_grads (gloo here, NCCL on
    the GPUs) and equal the 1-process full-batch gradients; dX gathers bitwise."""
    from oracle import lrs_backward as B
    port = _free_port()
    mp.spawn(_bwd_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    cfg = workloads.CONFIGS["c2_bf16"].replace(batch=5, in_h=6, in_w=6, c_in=16, c_out=24, rank_in=8, rank_out=8)
    inp = workloads.generate(cfg)
    dy = workloads.generate_dy(cfg, seed=4)
    ref = B.backward_factored(inp.x, dy, inp.u_in, inp.core, inp.u_out, inp.row_ptr, inp.col_idx, inp.values,
                              cfg.stride, cfg.pad)
    for k in ("d_u_in", "d_core", "d_u_out", "d_values"):
        got = np.load(tmp_path / f"{k}.npy")
        assert np.allclose(got, ref[k], rtol=1e-12, atol=1e-12), k
    assert np.array_equal(np.load(tmp_path / "dx.npy"), ref["dx"])
