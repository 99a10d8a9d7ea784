"""Host<->device copy rates on this box (pinned memory): H2D alone, D2H alone, both at once, by chunk size.
Sets the ceiling for the e2e leg (execute_host moves 16.8 MB in and 16.8 MB out per 2048^2 slice)."""
import time
import torch

dev = torch.device("cuda", 0)
GB = 1 << 30
h_in = torch.empty(2 * GB, dtype=torch.uint8).pin_memory()
h_out = torch.empty(2 * GB, dtype=torch.uint8).pin_memory()
d_in = torch.empty(2 * GB, dtype=torch.uint8, device=dev)
d_out = torch.empty(2 * GB, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunk, h2d=True, d2h=True, reps=2):
    n = (2 * GB) // chunk
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for i in range(n):
            sl = slice(i * chunk, (i + 1) * chunk)
            if h2d:
                with torch.cuda.stream(s1):
                    d_in[sl].copy_(h_in[sl], non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out[sl].copy_(d_out[sl], non_blocking=True)
    torch.cuda.synchronize()
    return 2 * GB * reps / (time.perf_counter() - t) / 1e9


for chunk_mb in (16, 64, 134, 256, 1024):
    c = chunk_mb << 20
    print(f"chunk {chunk_mb:5d} MB  H2D {run(c, True, False):6.1f} GB/s  D2H {run(c, False, True):6.1f} GB/s  "
          f"both {run(c, True, True):6.1f} GB/s each way")
