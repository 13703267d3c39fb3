"""Multi-GPU partitioning of the verify pass.

The pass shards along the two axes that need no exchange (suffix
copies never see each other and requests are independent):

* requests: rank r owns a contiguous block of requests;
* KV-head groups: when there are fewer request blocks than ranks, the ranks
  of one request block split its KV heads (and the q heads that read them).

Attention needs no collective.  The only exchange is one all-gather of the
per-prefix verdict results (scores, k*, accepted length) so every rank holds
the whole batch's selection — NCCL over NVLink on the GPU box, gloo in the
CPU tests.  This module is plumbing only: it computes index ranges and calls
torch.distributed; all arithmetic of the path runs in libparse.
"""

from __future__ import annotations

import dataclasses

import torch


@dataclasses.dataclass(frozen=True)
class ShardPlan:
    world: int
    rank: int
    n_req_groups: int
    n_head_groups: int
    req_offset: int       # first global request of this rank
    req_count: int
    kv_head_offset: int   # first KV head of this rank
    kv_head_count: int
    q_head_offset: int
    q_head_count: int

    @property
    def head_group(self) -> int:
        return self.rank % self.n_head_groups

    @property
    def owns_selection(self) -> bool:
        """The head-group-0 rank of a request block runs the readout for it."""
        return self.head_group == 0


def plan_shards(batch: int, num_q_heads: int, num_kv_heads: int, world: int, rank: int) -> ShardPlan:
    """Split `batch` requests x `num_kv_heads` KV heads over `world` ranks.

    Prefer pure request sharding; when world does not divide into the batch,
    use n_head_groups = the smallest divisor g of world with g | num_kv_heads
    and (world / g) | batch.  Raises if no such split exists.
    """
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    if num_q_heads % num_kv_heads:
        raise ValueError("num_q_heads must be a multiple of num_kv_heads")
    for g in range(1, world + 1):
        if world % g or num_kv_heads % g:
            continue
        n_req = world // g
        if batch % n_req:
            continue
        r = num_q_heads // num_kv_heads
        req_block, head_block = rank // g, rank % g
        per_req = batch // n_req
        per_kv = num_kv_heads // g
        return ShardPlan(world, rank, n_req, g, req_block * per_req, per_req, head_block * per_kv, per_kv,
                         head_block * per_kv * r, per_kv * r)
    raise ValueError(f"cannot split batch={batch} x kv_heads={num_kv_heads} over {world} ranks")


def local_views(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: ShardPlan, global_batch: bool = False):
    """Strided views of this rank's heads (and requests, if the tensors hold
    the global batch).  libparse accepts the strides directly, no copies."""
    if global_batch:
        sl = slice(plan.req_offset, plan.req_offset + plan.req_count)
        q, k, v = q[sl], k[sl], v[sl]
    qs = slice(plan.q_head_offset, plan.q_head_offset + plan.q_head_count)
    ks = slice(plan.kv_head_offset, plan.kv_head_offset + plan.kv_head_count)
    return q[:, :, qs], k[:, :, ks], v[:, :, ks]


def selection_buffers(batch: int, num_prefixes: int, device, want_stats: bool = True) -> dict:
    """Output buffers for parse_select_prefix laid out for one collective:
    accepted_len, k_star and scores are views of one contiguous int32 buffer
    `packed` = [accepted_len (b) | k_star (b) | scores (b x K, fp32 bits)], so
    gather_selection moves a rank's whole selection with a single all-gather."""
    b, K = batch, num_prefixes
    packed = torch.empty(b * (2 + K), dtype=torch.int32, device=device)
    return {
        "packed": packed,
        "accepted_len": packed[:b],
        "k_star": packed[b:2 * b],
        "scores": packed[2 * b:].view(torch.float32).view(b, K),
        "stats": torch.empty((b, 4), dtype=torch.int32, device=device) if want_stats else None,
        "status": torch.zeros(1, dtype=torch.int32, device=device),
    }


def gather_selection(local: dict, plan: ShardPlan, group=None) -> dict:
    """All-gather the per-request selection results of every rank.

    `local` holds this rank's accepted_len / k_star (int32 [b]) and scores
    (fp32 [b, K]) for its `req_count` requests.  Returns the same keys for
    the global batch, in request order (entries of head-group-0 ranks).
    """
    import torch.distributed as dist
    world = plan.world
    out = {}
    if "packed" in local:                 # one collective for the whole selection
        t = local["packed"]
        b, K = local["scores"].shape
        buf = torch.empty((world, t.numel()), dtype=t.dtype, device=t.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(buf, t, group=group)
        else:
            parts = list(buf.unbind(0))
            dist.all_gather(parts, t, group=group)
            buf = torch.stack(parts)
        keep = buf[[r for r in range(world) if r % plan.n_head_groups == 0]]
        out["accepted_len"] = keep[:, :b].reshape(-1)
        out["k_star"] = keep[:, b:2 * b].reshape(-1)
        out["scores"] = keep[:, 2 * b:].contiguous().view(torch.float32).reshape(-1, K)
        return out
    for key in ("accepted_len", "k_star", "scores"):
        t = local[key].contiguous()
        buf = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(buf, t, group=group)
        else:
            parts = list(buf.chunk(world))
            dist.all_gather(parts, t, group=group)
            buf = torch.cat(parts)
        # keep the head-group-0 rank of every request block, in request order
        per = t.shape[0]
        keep = [buf[r * per:(r + 1) * per] for r in range(world) if r % plan.n_head_groups == 0]
        out[key] = torch.cat(keep)
    return out


class PeerGather:
    """parse_select_prefix fused with the verdict all-gather over peer memory
    (`parse_select_prefix_allgather`): each rank's select kernel writes its
    requests' selection straight into every rank's gather buffer (NVLink P2P /
    CUDA IPC mappings) and returns once all ranks' slots have landed — one
    kernel instead of select + NCCL all-gather.

    Setup (once): every rank allocates its zeroed gather buffer, exports an IPC
    handle, and the handles are exchanged with `all_gather_object` (host
    plumbing over the process group); peers' buffers are mapped with
    `parse_peer_import`.  Calls must be made by all ranks in the same order."""

    def __init__(self, plan: ShardPlan, num_prefixes: int, device, group=None):
        import torch.distributed as dist
        from . import binding as bd
        self.bd = bd
        self.plan, self.K = plan, num_prefixes
        self.b = plan.req_count
        nbytes = bd.parse_peer_buffer_bytes(self.b, num_prefixes, plan.world)
        self.buf = torch.zeros((nbytes + 3) // 4, dtype=torch.int32, device=device)
        handle, offset = bd.parse_peer_export(self.buf.data_ptr())
        handles = [None] * plan.world
        dist.all_gather_object(handles, (handle, offset), group=group)
        ptrs, self.imported = [], []
        for r, (h, off) in enumerate(handles):
            if r == plan.rank:
                ptrs.append(self.buf.data_ptr())
            else:
                p = bd.parse_peer_import(h, off)
                ptrs.append(p)
                self.imported.append(p)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self.epoch = 0
        torch.cuda.synchronize(device)
        dist.barrier(group=group)          # every buffer is zeroed before any rank writes into it

    def __call__(self, logits: torch.Tensor, boundaries: torch.Tensor, threshold: float, **kw) -> dict:
        self.epoch += 1
        self.bd.parse_select_prefix_allgather(logits, boundaries, threshold, self.peers, self.plan.rank,
                                              self.plan.world, self.epoch, **kw)
        return self.results(self.epoch)

    def results(self, epoch: int) -> dict:
        """Views of the gathered selection of call `epoch`: valid until this rank's
        call epoch + 2 executes (three result sets; include/parse.h)."""
        b, K, world = self.b, self.K, self.plan.world
        slot = b * (2 + K)
        base = 256 // 4 + (epoch % 3) * world * slot
        sl = self.buf[base:base + world * slot].view(world, slot)
        if self.plan.n_head_groups > 1:
            sl = sl[[r for r in range(world) if r % self.plan.n_head_groups == 0]]
        return {"accepted_len": sl[:, :b].reshape(-1), "k_star": sl[:, b:2 * b].reshape(-1),
                "scores": sl[:, 2 * b:].reshape(-1).view(torch.float32).reshape(-1, K)}

    def close(self) -> None:
        for p in self.imported:
            self.bd.parse_peer_close(p)
        self.imported = []
