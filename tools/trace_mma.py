"""Merged MMA-side timeline of CTA 0 from a saved PARSE_TRACE trace
(TRACE_SAVE=... tools/trace_attn.py): per tile, each QK^T / PV group's issue
window and its completion (probe barrier timestamps), plus the softmax's S
loads and P hand-offs; and the tensor-pipe busy fraction implied by the
completions (512 cycles of MMA per group).

    python tools/trace_mma.py trace.npy [first_step] [n_steps]
"""
import sys

import numpy as np

tall = np.load(sys.argv[1])
j0 = int(sys.argv[2]) if len(sys.argv) > 2 else 40
nj = int(sys.argv[3]) if len(sys.argv) > 3 else 3
t = tall[:7 * 8192].reshape(7, 1024, 8)
sm = (t[0], t[1])
mm = (t[2], t[3])
ep = (t[5], t[6])
comp = [tall[57344 + 4096 * i: 57344 + 4096 * (i + 1)] for i in range(2)]
groups = []  # (tile, kind, step, issue_start, issue_end, done)
for i in range(2):
    m = mm[i]
    seq = []  # commit order: QK(0) at item start, then per step [QK(j+1)], PV(j)
    for j in range(1024):
        if m[j, 5] > 0:
            seq.append(("QK0", j, m[j, 5], m[j, 5]))
        if m[j, 4] > 0:
            seq.append(("QK", j + 1, m[j, 4], m[j, 7]))
        if m[j, 2] > 0:
            seq.append(("PV", j, m[j, 1], m[j, 2]))
    c = comp[i]
    for k, (kind, j, a, b) in enumerate(seq):
        groups.append((i, kind, j, a, b, c[k] if k < len(c) else 0))
done = np.array(sorted(g[5] for g in groups if g[5] > 0))
if len(done) > 8:
    span = done[-1] - done[0]
    print(f"groups completed: {len(done)}; implied tensor busy (512 cycles per group) over the span: "
          f"{512.0 * (len(done) - 1) / span:.3f}")
    gaps = np.diff(done)
    print(f"completion spacing: p10 {np.percentile(gaps, 10):.0f} p50 {np.median(gaps):.0f} p90 {np.percentile(gaps, 90):.0f}")
ev = []
for (i, kind, j, a, b, d) in groups:
    if j0 <= j < j0 + nj:
        nm = "QK" if kind != "PV" else "PV"
        ev.append((a, f"MMA{i} {nm}{i}({j}) issue start"))
        ev.append((b, f"MMA{i} {nm}{i}({j}) issued"))
        if d > 0:
            ev.append((d, f"      ==> {nm}{i}({j}) DONE"))
for i in range(2):
    for j in range(j0, j0 + nj):
        if sm[i][j, 1] > 0:
            ev.append((sm[i][j, 1], f"SMX{i} S({j}) ready"))
            ev.append((sm[i][j, 2], f"SMX{i} S({j}) loaded -> s_free"))
            ev.append((sm[i][j, 5], f"SMX{i} p_full({j})"))
        if ep[i][j, 5] > 0:
            ev.append((ep[i][j, 5], f"SMX{i} p_free wait start ({j})"))
            ev.append((ep[i][j, 6], f"SMX{i} p_free done ({j})"))
ev = [e for e in ev if e[0] > 0]
ev.sort()
b0 = ev[0][0] if ev else 0
for x, n in ev:
    print(f"{x - b0:7d}  {n}")

# Tensor-pipe occupancy model: every group is 8 MMAs of 64 cycles, executed in
# issue order; a group starts no earlier than its issue start and no earlier
# than the previous group's end, and cannot end before its last MMA was
# accepted (issue end) + 64.
allg = sorted((g for g in groups if g[3] > 0 and g[4] > 0), key=lambda g: g[4])
end = 0
idle = []
rows = []
for (i, kind, j, a, b, d) in allg:
    start = max(a, end, b - 448)
    if start > end and end > 0:
        idle.append(start - end)
    end = max(start + 512, b + 64)
    rows.append((i, kind, j, a, b, d, start, end))
if idle:
    tot = rows[-1][7] - rows[0][6]
    print(f"\nmodel: {len(rows)} groups, idle gaps {len(idle)}, idle {sum(idle)} of {tot} cycles "
          f"({sum(idle) / tot:.3f}); gap p50 {np.median(idle):.0f} p90 {np.percentile(idle, 90):.0f}")
    w0 = int(sys.argv[4]) if len(sys.argv) > 4 else len(rows) // 2
    print("tile kind step   issue_start issue_end  exec[start,end]  done  (idle before)")
    prev = None
    for r in rows[w0:w0 + 16]:
        gap = r[6] - prev if prev is not None else 0
        print(f"  {r[0]}  {r[1]:3s} {r[2]:4d}  {r[3]:10d} {r[4]:10d}  [{r[6]},{r[7]}] {r[5]}  ({gap})")
        prev = r[7]

# tile 0's QK^T(j+1): s_free seen -> first MMA accepted -> last MMA accepted -> commits done -> completion
m0 = mm[0]
rows = []
for j in range(1024):
    if m0[j, 4] > 0 and ep[0][j, 7] > 0 and ep[1][j, 7] > 0:
        rows.append((ep[0][j, 7] - m0[j, 4], ep[1][j, 7] - ep[0][j, 7], m0[j, 7] - ep[1][j, 7]))
if rows:
    r = np.array(rows)
    print(f"\nQK0 issue breakdown ({len(r)} groups): s_free seen -> 1st MMA accepted {np.median(r[:, 0]):.0f}, "
          f"1st -> 8th MMA {np.median(r[:, 1]):.0f}, 8th -> commits issued {np.median(r[:, 2]):.0f} (medians); "
          f"p90 {np.percentile(r[:, 0], 90):.0f} / {np.percentile(r[:, 1], 90):.0f} / {np.percentile(r[:, 2], 90):.0f}")
