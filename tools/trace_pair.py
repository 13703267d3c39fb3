"""Timeline of the CTA-pair kernel's cluster 0 (PARSE_TRACE build).

    PARSE_LIB=paper_2605_04263_b200/libparse_trace.so python tools/trace_pair.py --config qwen3_235b

Roles: 0 MMA (leader); 1/2 softmax WG0 rank 0/1; 3/4 softmax WG1 rank 0/1;
5/6 epilogue rank 0/1 (per item).  MMA per step: 0 before s_free, 1 s_free ok,
2 K/V landed, 3 QK issued, 4 before p_full, 5 P ready, 6 o_free ok.
Softmax per step: 0 before s_full, 1 S ready, 2 S loaded + s_free, 3 max
exchanged, 4 P packed, 5 p_empty ok (+rescale), 6 P stored + p_full.
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
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--g0", type=int, default=40)
ap.add_argument("--show", type=int, default=8)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
q, k, v = workloads.make_qkv(cfg, device="cuda", batch=a.batch)
bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
o = torch.empty_like(q)
tr = torch.zeros(7 * 1024 * 8, dtype=torch.int64, device="cuda")
os.environ["PARSE_TRACE_PTR"] = str(tr.data_ptr())
for _ in range(2):
    tr.zero_()
    pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, out=o)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(7, 1024, 8).astype(np.int64)
base = t[0, 0, 0]


def stat(name, d):
    d = d[(d > -1e8) & (d < 1e8)]
    if len(d):
        print(f"{name:44s} mean {d.mean():8.1f} p50 {np.median(d):8.1f} p90 {np.percentile(d, 90):8.1f}")


mm = t[0]
ok = (mm[:, 0] > 0) & (mm[1:].shape[0] > 0)
n = int(((mm[:, 3] > 0)).sum())
print("MMA steps", n)
st = mm[:n]
stat("MMA: wait s_free (1-0)", st[:, 1] - st[:, 0])
stat("MMA: wait K/V (2-1)", st[:, 2] - st[:, 1])
stat("MMA: QK issue (3-2)", st[:, 3] - st[:, 2])
stat("MMA: wait P (5-4)", st[:, 5] - st[:, 4])
stat("MMA: o_free (6-5)", st[:, 6] - st[:, 5])
stat("MMA: step period (QK issue to QK issue)", np.diff(st[:, 3]))
for r in range(1, 5):
    s = t[r]
    m = int((s[:, 6] > 0).sum())
    s = s[:m]
    print(f"-- softmax role {r} steps {m}")
    stat(" wait S (1-0)", s[:, 1] - s[:, 0])
    stat(" ld + s_free (2-1)", s[:, 2] - s[:, 1])
    stat(" mask/max/exchange (3-2)", s[:, 3] - s[:, 2])
    stat(" exp/pack (4-3)", s[:, 4] - s[:, 3])
    stat(" wait p_empty (5-4)", s[:, 5] - s[:, 4])
    stat(" P st + p_full (6-5)", s[:, 6] - s[:, 5])
    stat(" period", np.diff(s[:, 6]))
for r in (5, 6):
    s = t[r]
    m = int((s[:, 2] > 0).sum())
    s = s[:m]
    print(f"-- epilogue role {r} items {m}")
    stat(" wait o_full (1-0)", s[:, 1] - s[:, 0])
    stat(" drain O (2-1)", s[:, 2] - s[:, 1])
g0 = a.g0
print("timeline (cycles rel. to MMA step g0 event 0):")
ref = t[0, g0, 0]
for g in range(g0, g0 + a.show):
    print(g, "MMA", [int(x - ref) if x else None for x in t[0, g, :7]])
    for r in range(1, 5):
        print("   sm", r, [int(x - ref) if x else None for x in t[r, g, :7]])
