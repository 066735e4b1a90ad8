"""Run a few BP5 CG iterations (for ncu captures of the CG kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_07042_b200 as hx  # noqa: E402
from paper_2504_07042_b200 import solver as S  # noqa: E402

e = int(sys.argv[1]) if len(sys.argv) > 1 else 76
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
op = S.GlobalOperator(hx.box_mesh(e, e, e, 7), hx.KernelSpec("poisson", 1, "trilinear", 7), hx.SpectralBasis.build(7))
b = torch.randn(op.layout.n_local, dtype=torch.float64, device="cuda")
S.cg_solve(op, b, tol=0.0, max_iter=iters)
torch.cuda.synchronize()
