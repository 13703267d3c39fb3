"""Per-step timeline of the attention kernel's CTA 0 (PARSE_TRACE build).

    PARSE_LIB=paper_2605_04263_b200/libparse_trace.so python tools/trace_attn.py --config qwen3_235b

Softmax WG events (cycles): 0 before s_full wait, 1 S ready, 2 S in regs,
3 max done, 4 P stored, 5 p_full arrived.  MMA events per tile i: 0 before
p_full wait, 1 P ready, 2 PV+QK issued; step-level 6/7 around the KV waits.
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
ap.add_argument("--show", type=int, default=12)
ap.add_argument("--j0", type=int, default=10)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
B = a.batch or cfg.B
q, k, v = workloads.make_qkv(cfg, device="cuda", batch=B)
bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
o = torch.empty_like(q)
tr = torch.zeros(9 * 8192, dtype=torch.int64, device="cuda")
os.environ["PARSE_TRACE_PTR"] = str(tr.data_ptr())
for _ in range(2):
    tr.zero_()
    pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, out=o)
torch.cuda.synchronize()
tall = tr.cpu().numpy()
if os.environ.get("TRACE_SAVE"):
    np.save(os.environ["TRACE_SAVE"], tall)
t = tall[:7 * 8192].reshape(7, 1024, 8)
sm0, sm1, mm0, mm1, pr, ep0, ep1 = t[0], t[1], t[2], t[3], t[4], t[5], t[6]
t0 = min(x for x in (sm0[0, 0], sm1[0, 0], mm0[0, 0]) if x > 0)
n = int((sm0[:, 5] > 0).sum())
print(f"steps recorded: {n}")


def stats(name, arr):
    arr = arr[arr > 0]
    if len(arr):
        print(f"{name:40s} mean {arr.mean():8.1f}  p50 {np.median(arr):8.1f}  p90 {np.percentile(arr, 90):8.1f}"
              f"  p99 {np.percentile(arr, 99):8.1f}  sum {arr.sum():10.0f}")


for w, sm in (("WG0", sm0), ("WG1", sm1)):
    m = sm[:n]
    ok = (m[:, 0] > 0) & (m[:, 5] > 0)
    m = m[ok]
    stats(f"{w} wait for S (1-0)", m[:, 1] - m[:, 0])
    stats(f"{w} LDTM S (2-1)", m[:, 2] - m[:, 1])
    stats(f"{w} mask+max (3-2)", m[:, 3] - m[:, 2])
    stats(f"{w} exp+P store (4-3)", m[:, 4] - m[:, 3])
    e = (ep0 if w == "WG0" else ep1)[:n][ok]
    if (e[:, 5] > 0).any():
        sel = (e[:, 5] > 0) & (e[:, 6] > 0)
        stats(f"{w}   x+exp (ep5-3)", (e[:, 5] - m[:, 3])[sel])
        stats(f"{w}   p_free wait (ep6-ep5)", (e[:, 6] - e[:, 5])[sel])
        stats(f"{w}   pack+sum+P st (4-ep6)", (m[:, 4] - e[:, 6])[sel])
    stats(f"{w} rescale+arrive (5-4)", m[:, 5] - m[:, 4])
    stats(f"{w} softmax busy (5-1)", m[:, 5] - m[:, 1])
    stats(f"{w} period (0[j+1]-0[j])", np.diff(m[:, 0]))
for i, mm in ((0, mm0), (1, mm1)):
    m = mm[:n]
    stats(f"MMA tile{i} wait P (1-0)", m[:, 1] - m[:, 0])
    stats(f"MMA tile{i} issue PV+QK (2-1)", m[:, 2] - m[:, 1])
m = mm0[:n]
stats("MMA KV wait (7-6)", m[:, 7] - m[:, 6])
per = np.diff(m[:, 6])
stats("MMA step period", per)
per = per[per > 0]
for lo, hi in ((0, 2300), (2300, 3000), (3000, 5000), (5000, 1 << 40)):
    sel = (per >= lo) & (per < hi)
    print(f"   period in [{lo}, {hi}): {sel.sum():5d} steps, {per[sel].sum() / max(per.sum(), 1):.3f} of time")
p = pr[:n]
stats("producer wait K slot (1-0)", p[:, 1] - p[:, 0])
stats("producer wait V slot (3-2)", p[:, 3] - p[:, 2])
# lead: when K_{j+1}/V_j were issued vs when the MMA started waiting for them in step j
lead_v = mm0[1:n, 6] - pr[1:n, 3]
stats("V_j issued before MMA needs it", lead_v)
print("\nfirst steps (cycles rel. to start): WG0 S-ready / P-arrive | WG1 S-ready / P-arrive | MMA0 P-ready/issued | MMA1")
for j in range(min(a.show, n)):
    print(f"{j:3d}  {sm0[j,1]-t0:9d} {sm0[j,5]-t0:9d} | {sm1[j,1]-t0:9d} {sm1[j,5]-t0:9d} | "
          f"{mm0[j,1]-t0:9d} {mm0[j,2]-t0:9d} | {mm1[j,1]-t0:9d} {mm1[j,2]-t0:9d}")

# merged event timeline (cycles rel. to the first S-ready of the shown window)
names = {("sm", 0): "S wait", ("sm", 1): "S ready", ("sm", 2): "S regs", ("sm", 3): "max done", ("sm", 4): "P stored",
         ("sm", 5): "p_full arrive", ("sm", 6): "p_part arrive",
         ("mm", 0): "pre p_part wait", ("mm", 3): "p_part seen", ("mm", 4): "PVa issued", ("mm", 1): "p_full seen",
         ("mm", 2): "PVb+QK issued"}
j0 = a.j0
ev = []
for j in range(j0, j0 + 3):
    for w, sm in ((0, sm0), (1, sm1)):
        for e in range(7):
            if sm[j, e] > 0:
                ev.append((sm[j, e], f"j{j} WG{w} {names[('sm', e)]}"))
    for i, mm in ((0, mm0), (1, mm1)):
        for e in (0, 3, 4, 1, 2):
            if mm[j, e] > 0:
                ev.append((mm[j, e], f"j{j} MMA t{i} {names[('mm', e)]}"))
    ev.append((mm0[j, 6], f"j{j} MMA step start"))
    ev.append((mm1[j, 6], f"j{j} MMA V ready"))
    ev.append((mm0[j, 7], f"j{j} MMA K ready"))
ev.sort()
b0 = ev[0][0]
for t_, n_ in ev:
    print(f"{t_ - b0:8d}  {n_}")

# item transitions (tile 0): MMA item start / Q ready / K0 ready / first QK issued;
# softmax epilogue: before / after the o_full wait (recorded at the item's last step index + 1)
print("\nitem starts (MMA tile 0): step  start  q_ready  k0_ready  qk_issued   | WG0 epi o_full wait | WG0 S wait / S ready")
for j in range(min(a.show, n)):
    if pr[j, 4] > 0:
        print(f"{j:4d} {pr[j,4]-t0:9d} {pr[j,5]-t0:9d} {pr[j,6]-t0:9d} {pr[j,7]-t0:9d}   | "
              f"{sm0[j,6]-t0 if sm0[j,6] else 0:9d} {sm0[j,7]-t0 if sm0[j,7] else 0:9d} | {sm0[j,0]-t0:9d} {sm0[j,1]-t0:9d}")

# epilogue / item transition breakdown per softmax WG (indexed by the next item's first step):
# sm[.,6] before o_full wait, sm[.,7] o_full seen, ep 0 O stored, 2 before next_item, 3 item read, 4 row setup done,
# sm[next,0] S wait, sm[next,1] S ready
for w, sm, ep in (("WG0", sm0, ep0), ("WG1", sm1, ep1)):
    idx = [j for j in range(1, n) if ep[j, 3] > 0 and sm[j, 7] > 0 and sm[j, 1] > 0]
    if not idx:
        continue
    e = np.array([[sm[j, 7] - sm[j, 6], ep[j, 0] - sm[j, 7], ep[j, 2] - ep[j, 0], ep[j, 3] - ep[j, 2],
                   ep[j, 4] - ep[j, 3], sm[j, 0] - ep[j, 4], sm[j, 1] - sm[j, 0]] for j in idx])
    names_e = ["o_full wait", "O ld+cvt+store", "LSE", "next_item", "row setup", "to S wait", "S wait"]
    print(f"{w} item transitions ({len(idx)}): " + "  ".join(f"{nm} {v:.0f}" for nm, v in zip(names_e, e.mean(0))))
