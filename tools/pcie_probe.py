"""Host<->device copy ceilings of this box (pinned memory): H2D alone, D2H alone, both at once."""
import torch

dev = torch.device("cuda", 0)
n = 1 << 28  # 2 GiB of fp64
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device=dev)
d_b = torch.empty(n, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


gb = n * 8 / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D alone   {gb / t:6.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H alone   {gb / t:6.1f} GB/s")


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(both)
print(f"both        {gb / t:6.1f} GB/s each direction ({2 * gb / t:6.1f} combined)")
for chunks in (4, 16, 64):
    c = n // chunks

    def chunked():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        for i in range(chunks):
            with torch.cuda.stream(s1):
                d_a[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[i * c:(i + 1) * c].copy_(d_b[i * c:(i + 1) * c], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t = timed(chunked)
    print(f"both, {chunks:3d} chunks {gb / t:6.1f} GB/s each direction")
