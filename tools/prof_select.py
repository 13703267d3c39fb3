"""Launch parse_select_prefix a few times (for ncu) on a BASELINE config's readout."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04263_b200 as pb
import workloads
ap = argparse.ArgumentParser(); ap.add_argument("--config", default="long"); a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
lg = workloads.make_verdict_logits(cfg.B, cfg.K, seed=0, device="cuda", config_id=cfg.config_id)
bnd = torch.as_tensor(workloads.uniform_boundaries(cfg.N, cfg.K)).cuda()
out = None
for _ in range(4):
    out = pb.parse_select_prefix(lg, bnd, 0.985, aux_threshold=0.9, out=out)
torch.cuda.synchronize()
