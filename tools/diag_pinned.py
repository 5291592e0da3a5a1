"""Diagnostics: pinned host-buffer flavours vs PCIe copy rate on the GPU box
(torch pin_memory = cudaHostAlloc, vs 2 MB-aligned THP memory registered
with cudaHostRegister). Prints GB/s per direction, several trials each."""
import ctypes
import mmap
import time

import numpy as np
import torch

NB = 566 << 20


def thp_buffer(nbytes):
    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    libc.posix_memalign.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_size_t]
    libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    p = ctypes.c_void_p()
    size = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    assert libc.posix_memalign(ctypes.byref(p), 2 << 20, size) == 0
    libc.madvise(p, size, 14)  # MADV_HUGEPAGE
    arr = np.ctypeslib.as_array((ctypes.c_uint8 * size).from_address(p.value))
    arr[::4096] = 0  # first touch
    rc = torch.cuda.cudart().cudaHostRegister(p.value, size, 0)
    assert rc == 0 or int(rc) == 0, rc
    return torch.from_numpy(arr[:nbytes].view(np.float32))


def rate(dst, src, n=5):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return NB / min(ts) / 1e9, NB / (sum(ts) / n) / 1e9


def main():
    d = torch.empty(NB // 4, dtype=torch.float32, device="cuda")
    print("AnonHugePages before:", [l for l in open("/proc/meminfo") if "AnonHuge" in l or "Hugepagesize" in l])
    for trial in range(3):
        h = torch.empty(NB // 4, dtype=torch.float32, pin_memory=True)
        print(f"[pin_memory t{trial}] h2d best/mean {rate(d, h)} d2h {rate(h, d)}", flush=True)
        del h
        t = thp_buffer(NB)
        print(f"[thp+register t{trial}] h2d best/mean {rate(d, t)} d2h {rate(t, d)}", flush=True)
    print("AnonHugePages after:", [l for l in open("/proc/meminfo") if "AnonHuge" in l])
    print(open("/sys/kernel/mm/transparent_hugepage/enabled").read())


if __name__ == "__main__":
    main()
