"""PCIe ceiling of the box: concurrent H2D + D2H of contiguous pinned buffers, and the same with the
strided 2D shape stamg_sweep_host moves (rows of 16 KB at a 256 KB pitch)."""
import time
import torch
n = 1 << 29  # 4 GiB of doubles
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True); h_in.fill_(1.0)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d(); d2h()


gb = n * 8 / 1e9
print(f"contiguous 4 GiB: H2D {gb / run(h2d):.1f} GB/s, D2H {gb / run(d2h):.1f} GB/s, both at once {gb / run(both):.1f} GB/s each way")
# strided: 262144 rows of 2048 doubles (16 KB) out of rows of 32768 doubles (256 KB pitch): one chunk of 512 directions
rows, w, pitch = 16384, 2048, 32768
hbig = torch.empty(rows * pitch, dtype=torch.float64, pin_memory=True).view(rows, pitch)
hbig2 = torch.empty(rows * pitch, dtype=torch.float64, pin_memory=True).view(rows, pitch)
dch = torch.empty(rows, w, dtype=torch.float64, device="cuda")
dch2 = torch.ones(rows, w, dtype=torch.float64, device="cuda")


def both2d():
    with torch.cuda.stream(s1):
        dch.copy_(hbig[:, :w], non_blocking=True)
    with torch.cuda.stream(s2):
        hbig2[:, w:2 * w].copy_(dch2, non_blocking=True)


gb2 = rows * w * 8 / 1e9
print(f"strided rows of 16 KB at 256 KB pitch: both at once {gb2 / run(both2d):.1f} GB/s each way")
