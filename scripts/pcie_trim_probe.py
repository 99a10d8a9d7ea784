"""Does trimming the D2H of a 2048^2 image to the unit disk raise the e2e copy ceiling?
Pinned host memory; per chunk of 32 slices: H2D of the sinograms (contiguous) on one stream and, on
another, D2H of the images either whole or as per-band rectangles covering the disk (pixels with
r > 1 are exactly zero in every log-polar image), one cudaMemcpy3DAsync per band per chunk.
Prints slices/s for both and the trimmed byte fraction."""
import ctypes
import math
import time

import torch

n, nb, chunk, nchunks = 2048, 32, 32, 8
dev = torch.device("cuda", 0)
slice_bytes = n * n * 4
h_in = torch.empty((chunk * nchunks, n, n), dtype=torch.float32).pin_memory()
h_out = torch.empty((chunk * nchunks, n, n), dtype=torch.float32).pin_memory()
d_in = torch.empty((2, chunk, n, n), dtype=torch.float32, device=dev)
d_out = torch.empty((2, chunk, n, n), dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

# bands of rows with the column range covering every pixel centre inside the unit disk
c = n / 2
bands = []
rows_per = n // nb
tot = 0
for b in range(nb):
    r0, r1 = b * rows_per, (b + 1) * rows_per
    ymin = min(abs(-1 + (r + 0.5) * 2 / n) for r in range(r0, r1))
    if ymin > 1:
        continue
    half = math.sqrt(max(0.0, 1 - ymin * ymin))
    c0 = max(0, int(math.floor((-half + 1) * n / 2 - 0.5)) - 1)
    c1 = min(n, int(math.ceil((half + 1) * n / 2 - 0.5)) + 2)
    c0 &= ~3
    c1 = min(n, (c1 + 3) & ~3)
    bands.append((r0, r1, c0, c1))
    tot += (r1 - r0) * (c1 - c0)
frac = tot / (n * n)

cudart = ctypes.CDLL("libcudart.so.12") if False else None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        cudart = ctypes.CDLL(name)
        break
    except OSError:
        pass
if cudart is None:
    import glob, os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
    cudart = ctypes.CDLL(cands[0])


class Pitched(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("pitch", ctypes.c_size_t), ("xsize", ctypes.c_size_t), ("ysize", ctypes.c_size_t)]


class Pos(ctypes.Structure):
    _fields_ = [("x", ctypes.c_size_t), ("y", ctypes.c_size_t), ("z", ctypes.c_size_t)]


class Ext(ctypes.Structure):
    _fields_ = [("width", ctypes.c_size_t), ("height", ctypes.c_size_t), ("depth", ctypes.c_size_t)]


class Parms(ctypes.Structure):
    _fields_ = [("srcArray", ctypes.c_void_p), ("srcPos", Pos), ("srcPtr", Pitched), ("dstArray", ctypes.c_void_p),
                ("dstPos", Pos), ("dstPtr", Pitched), ("extent", Ext), ("kind", ctypes.c_int)]


def d2h_trim(dst_slice0, src, stream):
    for r0, r1, c0, c1 in bands:
        p = Parms()
        p.srcPtr = Pitched(src.data_ptr(), n * 4, n, n)
        p.srcPos = Pos(c0 * 4, r0, 0)
        p.dstPtr = Pitched(h_out[dst_slice0].data_ptr(), n * 4, n, n)
        p.dstPos = Pos(c0 * 4, r0, 0)
        p.extent = Ext((c1 - c0) * 4, r1 - r0, chunk)
        p.kind = 2  # cudaMemcpyDeviceToHost
        err = cudart.cudaMemcpy3DAsync(ctypes.byref(p), ctypes.c_void_p(stream.cuda_stream))
        assert err == 0, err


def run(trim, reps=2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for k in range(nchunks):
            sl = slice(k * chunk, (k + 1) * chunk)
            with torch.cuda.stream(s1):
                d_in[k & 1].copy_(h_in[sl], non_blocking=True)
            with torch.cuda.stream(s2):
                if trim:
                    d2h_trim(k * chunk, d_out[k & 1], s2)
                else:
                    h_out[sl].copy_(d_out[k & 1], non_blocking=True)
    torch.cuda.synchronize()
    return reps * nchunks * chunk / (time.perf_counter() - t)


# correctness of the band copy: every disk pixel arrives
d_out.normal_()
h_out.zero_()
d2h_trim(0, d_out[0], s2)
torch.cuda.synchronize()
yy, xx = torch.meshgrid(torch.arange(n), torch.arange(n), indexing="ij")
x = -1 + (xx + 0.5) * 2 / n
y = -1 + (yy + 0.5) * 2 / n
disk = (x * x + y * y) <= 1
ok = torch.equal(h_out[:chunk][:, disk], d_out[0].cpu()[:, disk])
print(f"bands {len(bands)}, trimmed D2H fraction {frac:.3f}, disk pixels all copied: {ok}")
for _ in range(2):
    full = run(False)
    trim = run(True)
    print(f"H2D + D2H whole images: {full:7.1f} slices/s   H2D + D2H disk bands: {trim:7.1f} slices/s  ({trim / full:.3f}x)")
