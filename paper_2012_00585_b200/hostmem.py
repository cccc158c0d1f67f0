"""Page-locked host buffers for the end-to-end path (fea_assemble_host* over PCIe).

torch's pinned allocator rounds every request up to a power of two (a 77 GB K buffer would
pin 128 GiB) and pins single-threaded. Here the pages are first touched by several threads,
then registered with cudaHostRegister, so config 5's K (77.3 GB) and values (32.7 GB) pin at
their own size. The registration is dropped when the array is garbage-collected.
"""
from __future__ import annotations

import os
import weakref
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def pinned_empty(shape, dtype=np.float64, threads: int | None = None) -> np.ndarray:
    import torch
    a = np.empty(shape, dtype)
    if a.nbytes == 0:
        return a
    flat = a.reshape(-1).view(np.uint8)
    threads = threads or min(32, os.cpu_count() or 1)
    step = max(1 << 26, (flat.size + threads - 1) // threads)
    with ThreadPoolExecutor(threads) as ex:  # first touch in parallel (numpy fill drops the GIL)
        list(ex.map(lambda o: flat[o:o + step].fill(0), range(0, flat.size, step)))
    cudart = torch.cuda.cudart()
    ptr = a.ctypes.data
    err = cudart.cudaHostRegister(ptr, a.nbytes, 0)
    if int(err) != 0:
        raise RuntimeError(f"cudaHostRegister({a.nbytes} bytes) failed: {int(err)}")
    weakref.finalize(a, cudart.cudaHostUnregister, ptr)
    return a
