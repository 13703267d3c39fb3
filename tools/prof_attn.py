"""Launch parse_verify_attn a few times on one BASELINE config (for ncu).

    ncu --metrics sm__cycles_elapsed.avg,... -k regex:attn_sm100 -s 2 -c 1 \
        python tools/prof_attn.py --config qwen3_235b
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_04263_b200 as pb  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen3_235b")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--fp8", action="store_true", help="time the FP8 (e4m3) variant")
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
B = a.batch or cfg.B
q, k, v = workloads.make_qkv(cfg, device="cuda", batch=B)
bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
tree = workloads.make_tree_parent(cfg.S, seed=workloads.seed_for(cfg.config_id, 0, "tree")) if cfg.tree else None
o = torch.empty_like(q)
if a.fp8:
    (q8, sq), (k8, sk), (v8, sv) = workloads.to_e4m3(q), workloads.to_e4m3(k), workloads.to_e4m3(v)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.iters)]
for i in range(a.iters):
    ev[2 * i].record()
    if a.fp8:
        pb.parse_verify_attn_fp8(q8, k8, v8, sq, sk, sv, bnd, cfg.K, cfg.S, tree_parent=tree, out=o)
    else:
        pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree, out=o)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
print("ms per call:", [round(ev[2 * i].elapsed_time(ev[2 * i + 1]), 3) for i in range(a.iters)])
