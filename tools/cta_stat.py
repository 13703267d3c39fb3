"""Per-CTA accounting of the attention kernel (PARSE_CTASTAT build): how much
of the kernel's span each persistent CTA spends busy, and how its busy time
compares with the tensor-pipe time of the tile-steps it ran (1024 cycles per
128x128 tile-step at D=128 bf16: 16 MMAs of ~64 cycles).

    PARSE_LIB=paper_2605_04263_b200/libparse_ctastat.so python tools/cta_stat.py --config long --batch 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04263_b200 as pb  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen3_235b")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--step-cycles", type=float, default=1024.0)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
B = a.batch or cfg.B
q, k, v = workloads.make_qkv(cfg, device="cuda", batch=B)
bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
tree = workloads.make_tree_parent(cfg.S, seed=workloads.seed_for(cfg.config_id, 0, "tree")) if cfg.tree else None
o = torch.empty_like(q)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
tr = torch.zeros(nsm * 8, dtype=torch.int64, device="cuda")
os.environ["PARSE_TRACE_PTR"] = str(tr.data_ptr())
for _ in range(3):
    tr.zero_()
    pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree, out=o)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(nsm, 8)
t = t[t[:, 1] > 0]
ns0, ns1, c0, c1, s0, s1, items = (t[:, i].astype(np.float64) for i in range(7))
span_ns = ns1.max() - ns0.min()
clk_per_ns = np.median((c1 - c0) / (ns1 - ns0))
busy = c1 - c0
steps = s0 + s1
eff = steps * a.step_cycles / busy
tail_ns = ns1.max() - ns1
print(f"{a.config} B={B}: CTAs {len(t)}  span {span_ns / 1e3:.1f} us  clock {clk_per_ns:.3f} GHz")
print(f"  tile-steps total {steps.sum():.0f}  per CTA mean {steps.mean():.0f} min {steps.min():.0f} max {steps.max():.0f}")
print(f"  items per CTA mean {items.mean():.1f}  steps/item {steps.sum() / items.sum():.1f}")
print(f"  busy/span  mean {(busy / clk_per_ns).mean() / span_ns:.4f}")
print(f"  in-CTA tensor efficiency (steps*{a.step_cycles:.0f}/busy) mean {eff.mean():.4f} min {eff.min():.4f} max {eff.max():.4f}")
print(f"  start skew max {(ns0.max() - ns0.min()) / 1e3:.2f} us   tail (max end - end) mean {tail_ns.mean() / 1e3:.2f} us max {tail_ns.max() / 1e3:.2f} us")
print(f"  overall = steps*{a.step_cycles:.0f} / (CTAs*span) = {steps.sum() * a.step_cycles / (len(t) * span_ns * clk_per_ns):.4f}")
