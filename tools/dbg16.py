import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2403_01136_b200 import qweight
dev = torch.device('cuda:0')
for (n, k) in ((7168, 28672), (1024, 28672), (7168, 4096), (7168, 8192), (512, 1024)):
    w = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    x = (torch.randn(32, k, device=dev) + 0.05).to(torch.bfloat16)
    qw = qweight.quantize(w, 16)
    ref = x.float() @ w.float().T
    for rep in range(2):
        got = qweight.qlinear(qw, x, phase=1).float()
        bad = ~torch.isfinite(got)
        e = float((got - ref).abs().nan_to_num(1e9).max() / ref.abs().max())
        print(n, k, rep, "nonfinite", int(bad.sum()), "err", e, "bad rows", torch.nonzero(bad.any(0)).flatten()[:8].tolist(), "bad toks", torch.nonzero(bad.any(1)).flatten()[:8].tolist(), flush=True)
