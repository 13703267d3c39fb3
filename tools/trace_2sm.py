"""Timeline of the 2-SM kernel's first cluster (PARSE_TRACE build, PARSE_2SM=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04263_b200 as pb  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "qwen3_235b"]
q, k, v = workloads.make_qkv(cfg, device="cuda")
bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
o = torch.empty_like(q)
tr = torch.zeros(3 * 1024 * 8, dtype=torch.int64, device="cuda")
os.environ["PARSE_TRACE_PTR"] = str(tr.data_ptr())
for _ in range(2):
    tr.zero_()
    pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, out=o)
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(3, 1024, 8)
mm, s0, s1 = t[0], t[1], t[2]
t0 = s0[0, 0]
names = {(0, 0): "MMA p_part seen", (0, 1): "MMA PVa issued", (0, 2): "MMA p_full seen", (0, 3): "MMA PVb issued",
         (0, 4): "MMA QK(j+2) issued", (1, 0): "SM0 S wait", (1, 1): "SM0 S ready", (1, 2): "SM0 max done",
         (1, 3): "SM0 p_part", (1, 4): "SM0 p_full", (2, 0): "SM1 S wait", (2, 1): "SM1 S ready", (2, 2): "SM1 max done",
         (2, 3): "SM1 p_part", (2, 4): "SM1 p_full"}
for name, arr in (("SM0", s0), ("SM1", s1)):
    ok = (arr[:, 1] > 0) & (arr[:, 4] > 0)
    a = arr[ok]
    print(name, "steps", ok.sum(), "S wait", np.median(a[:, 1] - a[:, 0]), "S->max", np.median(a[:, 2] - a[:, 1]),
          "max->p_part", np.median(a[:, 3] - a[:, 2]), "p_part->p_full", np.median(a[:, 4] - a[:, 3]),
          "period", np.median(np.diff(a[:, 1])))
ev = []
for j in range(20, 24):
    for role, arr in ((0, mm), (1, s0), (2, s1)):
        for e in range(5):
            if arr[j, e] > 0:
                ev.append((arr[j, e] - t0, f"j{j} {names[(role, e)]}"))
for tt, n in sorted(ev):
    print(f"{tt:9d} {n}")
