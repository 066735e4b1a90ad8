import time, torch, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2504_07042_b200 as hx
dev = torch.device("cuda", 0)
t0 = time.perf_counter(); mesh = hx.box_mesh(128, 128, 96, 7, perturbation=0.1, seed=0); t1 = time.perf_counter()
print(f"box_mesh {t1-t0:.3f} s")
b = hx.SpectralBasis.build(7)
for src in ("trilinear", "stored", "trilinear-partial", "parallelepiped"):
    m = mesh if src != "parallelepiped" else hx.box_mesh(128, 128, 96, 7)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    op = hx.LocalOperator(hx.KernelSpec("poisson", 1, src, 7), m, b, device=dev)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"setup {src:18s} {t1-t0:.3f} s")
    del op; torch.cuda.empty_cache()
