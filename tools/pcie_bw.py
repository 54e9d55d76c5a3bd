"""Host<->device copy bandwidth for the e2e path's per-step transfers (25 MB
each way at 1,048,576 particles): pinned vs write-combined host memory, one
vs several concurrent streams."""
import ctypes
import time

import numpy as np
import torch

n = 3 * 1_048_576
nbytes = n * 8
cudart = ctypes.CDLL("libcudart.so")
for lib_name in ("libcudart.so.12", "libcudart.so"):
    try:
        cudart = ctypes.CDLL(lib_name)
        break
    except OSError:
        pass


def host_alloc(flags):
    p = ctypes.c_void_p()
    assert cudart.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(nbytes), ctypes.c_uint(flags)) == 0
    return p


d = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
cudart.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]


def run(host, kind, nstreams):
    per = nbytes // nstreams
    def go():
        for k in range(nstreams):
            off = k * per
            size = per if k < nstreams - 1 else nbytes - off
            s = streams[k]
            if kind == 1:   # H2D
                cudart.cudaMemcpyAsync(ctypes.c_void_p(d.data_ptr() + off), ctypes.c_void_p(host.value + off), size, 1, ctypes.c_void_p(s.cuda_stream))
            else:
                cudart.cudaMemcpyAsync(ctypes.c_void_p(host.value + off), ctypes.c_void_p(d.data_ptr() + off), size, 2, ctypes.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
    go()
    best = 1e9
    for _ in range(15):
        t = time.perf_counter()
        go()
        best = min(best, time.perf_counter() - t)
    return best


for flags, name in ((0, "pinned"), (4, "write-combined"), (1, "portable")):
    h = host_alloc(flags)
    for kind, kname in ((1, "H2D"), (2, "D2H")):
        for ns in (1, 2, 4):
            t = run(h, kind, ns)
            print(f"{name:15s} {kname} streams={ns}: {t * 1e3:.3f} ms  {nbytes / t / 1e9:.1f} GB/s")

# torch's pin_memory() allocation, copied with cudaMemcpyAsync (the e2e path's
# HostParticleSet memory) and with torch's own copy_
t = torch.zeros(n, dtype=torch.float64).pin_memory()
class _P:
    value = t.data_ptr()
for kind, kname in ((1, "H2D"), (2, "D2H")):
    tt = run(_P, kind, 1)
    print(f"torch pin_memory via cudaMemcpyAsync {kname}: {tt * 1e3:.3f} ms  {nbytes / tt / 1e9:.1f} GB/s")
for name, fn in (("H2D", lambda: d.copy_(t, non_blocking=True)), ("D2H", lambda: t.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(15):
        a = time.perf_counter(); fn(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - a)
    print(f"torch pin_memory via copy_ {name}: {best * 1e3:.3f} ms  {nbytes / best / 1e9:.1f} GB/s")
