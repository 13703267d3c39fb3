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
names = {(0, 0): "MMA s_used seen", (0, 1): "MMA K ready", (0, 2): "MMA QK issued", (0, 3): "MMA p_full seen",
         (0, 4): "MMA PV issued"}
for r_ in (1, 2):
    for e_, n_ in enumerate(["S wait", "S ready", "s_used arrived", "exps done", "p_empty ok", "p_full arrived"]):
        names[(r_, e_)] = f"SM{r_ - 1} {n_}"
for name, arr in (("SM0", s0), ("SM1", s1)):
    ok = (arr[:, 1] > 0) & (arr[:, 5] > 0)
    a = arr[ok]
    print(name, "steps", ok.sum(), "S wait", np.median(a[:, 1] - a[:, 0]), "S->s_used", np.median(a[:, 2] - a[:, 1]),
          "->exps done", np.median(a[:, 3] - a[:, 2]), "p_empty wait", np.median(a[:, 4] - a[:, 3]),
          "store+arrive", np.median(a[:, 5] - a[:, 4]), "period", np.median(np.diff(a[:, 1])))
ev = []
for j in range(20, 24):
    for role, arr in ((0, mm), (1, s0), (2, s1)):
        for e in range(6):
            if arr[j, e] > 0:
                ev.append((arr[j, e] - t0, f"j{j} {names[(role, e)]}"))
for tt, n in sorted(ev):
    print(f"{tt:9d} {n}")
