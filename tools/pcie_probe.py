"""PCIe copy bandwidth on the box: pinned H2D, D2H, and both directions at once (the
bound of bench.py's e2e, which moves every request's inputs in and outputs out)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05288_b200 as D  # noqa: E402

L = D.lib()
n = 1 << 30
h1, h2, d1, d2 = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
s1, s2 = C.c_void_p(), C.c_void_p()
for s in (s1, s2):
    L.disc_cuda_stream_create(C.byref(s))
L.disc_cuda_host_alloc(n, C.byref(h1))
L.disc_cuda_host_alloc(n, C.byref(h2))
L.disc_cuda_malloc(n, s1, C.byref(d1))
L.disc_cuda_malloc(n, s1, C.byref(d2))
L.disc_cuda_device_synchronize()


def run(h2d, d2h, reps=3):
    L.disc_cuda_device_synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            L.disc_cuda_memcpy(d1, h1, n, 0, s1)
        if d2h:
            L.disc_cuda_memcpy(h2, d2, n, 1, s2)
    L.disc_cuda_device_synchronize()
    return (h2d + d2h) * n * reps / (time.perf_counter() - t) / 1e9


run(1, 1, 1)
print(f"H2D {run(1, 0):.1f} GB/s  D2H {run(0, 1):.1f} GB/s  both {run(1, 1):.1f} GB/s (sum of directions)")
