"""Time parse_verify_attn (plan path: counter memset + kernel) on BASELINE
configs with CUDA events and print ms / TFLOP/s per config.  PARSE_LIB picks
a library variant (A/B).

    python tools/time_attn.py qwen3_235b qwen3_8b [--batch B] [--iters 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_04263_b200 as pb  # noqa: E402
import workloads  # noqa: E402
from bench import visible_pairs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
for name in a.configs:
    cfg = workloads.CONFIGS[name]
    B = a.batch or min(cfg.B, 16)
    q, k, v = workloads.make_qkv(cfg, device="cuda", batch=B)
    bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
    tree = workloads.make_tree_parent(cfg.S, seed=workloads.seed_for(cfg.config_id, 0, "tree")) if cfg.tree else None
    o = torch.empty_like(q)
    plan = pb.VerifyAttnPlan(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree, out=o)
    for _ in range(3):
        plan.run(q, k, v, o)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.iters):
        plan.run(q, k, v, o)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    flops = 4.0 * cfg.d * cfg.Hq * visible_pairs(cfg, bnd, tree) * B
    print(json.dumps({"config": name, "B": B, "ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1),
                      "lib": os.environ.get("PARSE_LIB", "libparse.so")}), flush=True)
    plan.close()
    del q, k, v, o
    torch.cuda.empty_cache()
