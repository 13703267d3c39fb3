"""Multi-GPU sharding invariant on one GPU (SURVEY §8 e): every shard of
`plan_shards` — a block of requests and/or a KV-head group, passed to
libparse as strided views without copies — produces outputs bitwise equal to
the same rows / heads of the unsharded pass, and the per-shard selections
reassemble the unsharded selection.  (The kernel's work items never mix
requests or KV groups, so sharding cannot change any arithmetic.)"""

import numpy as np
import pytest
import torch

import paper_2605_04263_b200 as pb
import workloads
from paper_2605_04263_b200.parallel import local_views, plan_shards

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_shards_bitwise_equal_unsharded(world):
    # config-3 head geometry (64 q / 4 kv heads), shorter draft; B=2 < world forces KV-head-group shards
    cfg = workloads.Config("shard", 61, 2, 64, 4, 128, 1024, 8, 32)
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    q, k, v = workloads.make_qkv(cfg, device="cuda")
    full, full_lse = pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, want_lse=True)
    lg = workloads.make_verdict_logits(cfg.B, cfg.K, seed=5, config_id=61).cuda()
    bnd_d = torch.as_tensor(bnd).cuda()
    full_sel = pb.parse_select_prefix(lg, bnd_d, 0.985)
    torch.cuda.synchronize()
    got_acc = torch.empty_like(full_sel["accepted_len"])
    for rank in range(world):
        plan = plan_shards(cfg.B, cfg.Hq, cfg.Hkv, world, rank)
        ql, kl, vl = local_views(q, k, v, plan, global_batch=True)
        o, lse = pb.parse_verify_attn(ql, kl, vl, bnd, cfg.K, cfg.S, want_lse=True)
        torch.cuda.synchronize()
        rs = slice(plan.req_offset, plan.req_offset + plan.req_count)
        hs = slice(plan.q_head_offset, plan.q_head_offset + plan.q_head_count)
        assert torch.equal(o, full[rs, :, hs]), (world, rank)
        assert torch.equal(lse, full_lse[rs, hs]), (world, rank)
        if plan.owns_selection:
            sel = pb.parse_select_prefix(lg[rs], bnd_d, 0.985)
            got_acc[rs] = sel["accepted_len"]
    torch.cuda.synchronize()
    assert torch.equal(got_acc, full_sel["accepted_len"])
    assert np.array_equal(got_acc.cpu().numpy(), full_sel["accepted_len"].cpu().numpy())
