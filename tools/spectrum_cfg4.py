"""Print the spectrum of config 4's M = T'(C'C)T (top-k eig subproblem) in fp64 torch."""
import numpy as np
import torch

import bench_configs as bc
import paper_1505_07570_b200 as rn

n, d, c, k, comps = 131072, 64, 2048, 64, 16
g = bc.gen(bc.data_seed(4))
means = 3.0 * torch.randn(comps, d, device="cuda", generator=g)
lab = torch.randint(0, comps, (n,), device="cuda", generator=g)
X = (means[lab] + torch.randn(n, d, device="cuda", generator=g)).float().contiguous()
sub = X[torch.from_numpy(rn.sample_without_replacement(n, 4096, rn.derive_seed(bc.op_seed(4), 3))).cuda()].double()
dd = torch.cdist(sub, sub)
iu = torch.triu_indices(4096, 4096, 1, device="cuda")
sigma = float(torch.median(dd[iu[0], iu[1]]).item())
sel = torch.from_numpy(rn.sample_without_replacement(n, c, rn.derive_seed(bc.op_seed(4), 1)).astype(np.int64)).cuda()
x = X.double()
xs = x[sel]
sq = (x * x).sum(1)
sqs = (xs * xs).sum(1)
C = torch.exp((x @ xs.T - 0.5 * (sq[:, None] + sqs[None, :])) / sigma**2)
W = C[sel]
lw, vw = torch.linalg.eigh(0.5 * (W + W.T))
lw, vw = lw.flip(0), vw.flip(1)
floor = np.finfo(np.float64).eps * float(lw[0]) * n
kp = int((lw > floor).sum())
T = vw[:, :kp] / lw[:kp].sqrt()
M = T.T @ (C.T @ C) @ T
lm = torch.linalg.eigvalsh(0.5 * (M + M.T)).flip(0).cpu().numpy()
print("sigma", sigma, "kept", kp, "W lam max/min", float(lw[0]), float(lw[-1]))
for i in (1, 2, 8, 16, 32, 63, 64, 65, 96, 128, 129, 160, 192, 256, 512, 1024, kp):
    print(f"lam_M[{i}] = {lm[i - 1]:.6e}  ratio to lam_64 {lm[i - 1] / lm[63]:.4e}")
