"""Small calls of every libparse entry point, for compute-sanitizer
(memcheck / racecheck / synccheck) on the B200:
   compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_04263_b200 as pb  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.Config("san", 991, 2, 8, 2, 128, 300, 5, 16)
bnd = np.array([0, 40, 150, 299, 300], np.int32)
q, k, v = workloads.make_qkv(cfg, device="cuda")
o, lse = pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, want_lse=True)
o32, _ = pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, precision=pb.PARSE_PREC_FP32_DEBUG)
(q8, sq), (k8, sk), (v8, sv) = workloads.to_e4m3(q), workloads.to_e4m3(k), workloads.to_e4m3(v)
o8, _ = pb.parse_verify_attn_fp8(q8, k8, v8, sq, sk, sv, bnd, cfg.K, cfg.S)
tree = workloads.make_tree_parent(16, seed=3)
ot, _ = pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S, tree_parent=tree)
# several items per CTA, one- and two-tile items interleaved (r = 3): the
# one-S-buffer protocol across item boundaries and its dummy S uses
cm = workloads.Config("san_mixed", 992, 4, 12, 4, 128, 1024, 9, 32)
bm = np.sort(np.random.default_rng(5).integers(0, 1025, 9)).astype(np.int32)
qm, km, vm = workloads.make_qkv(cm, device="cuda")
om, _ = pb.parse_verify_attn(qm, km, vm, bm, cm.K, cm.S, want_lse=True)
del qm, km, vm, om
# ragged + paged
rb = workloads.make_ragged_batch([300, 77, 129], 8, 2, 128, 16, 40, page_size=16, device="cuda", keep_lists=False)
ov, _ = pb.parse_verify_attn_varlen(rb.q, rb.k, rb.v, rb.Ns, rb.Ks, rb.boundaries, 16, row_offsets=rb.row_offsets,
                                    block_table=rb.block_table.cuda(), page_size=16)
lg = workloads.make_verdict_logits(2, cfg.K, seed=1).cuda()
sel = pb.parse_select_prefix(lg, torch.as_tensor(bnd).cuda(), 0.985)
plan = pb.VerifyAttnPlan(q, k, v, bnd, cfg.K, cfg.S, out=torch.empty_like(q))
plan.run(q, k, v, plan_out := torch.empty_like(q))
h = torch.randn(2, cfg.K, 512, device="cuda").to(torch.bfloat16)
g = torch.randn(512, device="cuda").to(torch.bfloat16)
wu = torch.randn(2, 512, device="cuda").to(torch.bfloat16)
vl = pb.parse_verdict_logits(h, g, wu)
vs = pb.parse_verdict_select(h, g, wu, torch.as_tensor(np.sort(np.random.default_rng(2).integers(0, 300, h.shape[1]))
                                                       .astype(np.int32)).cuda(), 0.7)
z = torch.randn(2, cfg.K, 1000, device="cuda").to(torch.bfloat16)
ro = pb.parse_vocab_readout(z, 3, 7)
torch.cuda.synchronize()
print("sanitize run ok")
