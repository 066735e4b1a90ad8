"""Per-kernel device-time breakdown of BP5 CG iterations (torch profiler / CUPTI)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07042_b200 as hx  # noqa: E402
from paper_2504_07042_b200 import solver as S  # noqa: E402

e = int(sys.argv[1]) if len(sys.argv) > 1 else 76
src = sys.argv[2] if len(sys.argv) > 2 else "trilinear"
mesh = hx.box_mesh(e, e, e, 7)
op = S.GlobalOperator(mesh, hx.KernelSpec("poisson", 1, src, 7), hx.SpectralBasis.build(7))
b = torch.randn(op.layout.n_local, dtype=torch.float64, device="cuda")
S.cg_solve(op, b, tol=0.0, max_iter=3)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    S.cg_solve(op, b, tol=0.0, max_iter=10)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20, max_name_column_width=60))
