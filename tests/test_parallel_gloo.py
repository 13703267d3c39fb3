"""world_size-2 (and 4) gloo tests of the multi-GPU plumbing on CPU: shard
planning covers every (request, head) exactly once, and the verdict
all-gather reassembles the single-process result.  The per-rank compute here
is the oracle (test-only stand-in for the GPU kernels, which need a B200)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2605_04263_b200.parallel import gather_selection, local_views, plan_shards, selection_buffers
import workloads


@pytest.mark.parametrize("B,Hq,Hkv,world", [(16, 64, 4, 8), (2, 64, 4, 8), (8, 32, 8, 4), (3, 4, 2, 6), (64, 64, 4, 8)])
def test_plan_covers_every_request_head_once(B, Hq, Hkv, world):
    seen = np.zeros((B, Hq), dtype=int)
    for rank in range(world):
        p = plan_shards(B, Hq, Hkv, world, rank)
        assert p.q_head_count == p.kv_head_count * (Hq // Hkv)
        seen[p.req_offset:p.req_offset + p.req_count, p.q_head_offset:p.q_head_offset + p.q_head_count] += 1
        # q heads of the shard read only the shard's kv heads
        r = Hq // Hkv
        assert p.q_head_offset // r == p.kv_head_offset
    assert (seen == 1).all()


def test_plan_rejects_impossible_split():
    with pytest.raises(ValueError):
        plan_shards(3, 4, 1, 2, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, K, result_path, packed=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = plan_shards(B, 8, 2, world, rank)
        # every rank generates only its own requests (same per-request seeds as 1 rank)
        lg = workloads.make_verdict_logits(plan.req_count, K, seed=0, batch_offset=plan.req_offset, config_id=7)
        bnd = workloads.uniform_boundaries(400, K)
        sel = oracle.select_prefix(lg.double().numpy(), bnd, 0.985)
        local = {"accepted_len": torch.from_numpy(sel["accepted_len"]), "k_star": torch.from_numpy(sel["k_star"]),
                 "scores": torch.from_numpy(sel["scores"])}
        if packed:      # the bench layout: one buffer, one collective
            buf = selection_buffers(plan.req_count, K, "cpu")
            for key in ("accepted_len", "k_star", "scores"):
                buf[key].copy_(local[key])
            local = buf
        full = gather_selection(local, plan)
        if rank == 0:
            torch.save(full, result_path)
        # head-sharded attention views: shapes consistent with the plan
        cfg = workloads.Config("gloo", 8, plan.req_count, 8, 2, 64, 40, 2, 4)
        q, k, v = workloads.make_qkv(cfg, batch_offset=plan.req_offset)
        ql, kl, vl = local_views(q, k, v, plan)
        assert ql.shape[2] == plan.q_head_count and kl.shape[2] == plan.kv_head_count
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,B,packed", [(2, 6, False), (4, 2, False), (2, 6, True), (4, 2, True)])
def test_gather_matches_single_process(tmp_path, world, B, packed):
    K = 10
    path = str(tmp_path / "full.pt")
    mp.spawn(_worker, args=(world, _free_port(), B, K, path, packed), nprocs=world, join=True)
    full = torch.load(path)
    lg = workloads.make_verdict_logits(B, K, seed=0, config_id=7)
    want = oracle.select_prefix(lg.double().numpy(), workloads.uniform_boundaries(400, K), 0.985)
    assert np.array_equal(full["accepted_len"].numpy(), want["accepted_len"])
    assert np.array_equal(full["k_star"].numpy(), want["k_star"])
    assert np.array_equal(full["scores"].numpy(), want["scores"])
