import sys; sys.path.insert(0, '/root/repo')
import torch, workloads, paper_2605_04263_b200 as pb
cfg = workloads.CONFIGS["tiny"]
bnd = workloads.uniform_boundaries(cfg.N, cfg.K)
q, k, v = workloads.make_qkv(cfg, device="cuda")
o, _ = pb.parse_verify_attn(q, k, v, bnd, cfg.K, cfg.S)
torch.cuda.synchronize()
print("ok", o.float().abs().max().item())
