"""GPU test of the fused select + peer all-gather (parse_select_prefix_allgather,
SURVEY §8 e): world_size 2 and 3 processes sharing cuda:0 map each other's
gather buffers over CUDA IPC; after each call every rank's buffer must hold
the whole batch's selection, equal (bit-exact: k*, accepted length; scores to
2 fp32 ulp) to the fp64 oracle on the same seeded logits, over several calls
(both buffer sets, rising epochs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, K, calls, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2605_04263_b200 as pb
        from paper_2605_04263_b200.parallel import PeerGather, plan_shards
        torch.cuda.set_device(0)
        plan = plan_shards(B, 8, 2, world, rank)
        pg = PeerGather(plan, K, "cuda")
        bnd = torch.as_tensor(workloads.uniform_boundaries(400, K)).cuda()
        for c in range(calls):
            lg = workloads.make_verdict_logits(plan.req_count, K, seed=c, batch_offset=plan.req_offset,
                                               config_id=11).cuda()
            res = pg(lg, bnd, 0.985)
            torch.cuda.synchronize()
            torch.save({k: v.cpu() for k, v in res.items()}, os.path.join(out_dir, f"r{rank}_c{c}.pt"))
        dist.barrier()
        pg.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,B", [(2, 6), (3, 3)])
def test_peer_gather_matches_oracle(tmp_path, world, B):
    K, calls = 37, 5
    mp.spawn(_worker, args=(world, _free_port(), B, K, calls, str(tmp_path)), nprocs=world, join=True)
    bnd = workloads.uniform_boundaries(400, K)
    for c in range(calls):
        lg = workloads.make_verdict_logits(B, K, seed=c, config_id=11)
        want = oracle.select_prefix(lg.double().numpy(), bnd, 0.985)
        for r in range(world):
            got = torch.load(os.path.join(tmp_path, f"r{r}_c{c}.pt"))
            assert np.array_equal(got["accepted_len"].numpy(), want["accepted_len"]), (c, r)
            assert np.array_equal(got["k_star"].numpy(), want["k_star"]), (c, r)
            sc = got["scores"].numpy().astype(np.float64)
            ulp = np.spacing(np.abs(want["scores"]).astype(np.float32)).astype(np.float64)
            assert (np.abs(sc - want["scores"]) <= 2 * ulp + 1e-30).all(), (c, r)
