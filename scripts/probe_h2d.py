"""H2D bandwidth probe: DMA copies of entry-activation-sized chunks from pinned memory (development aid)."""
import time

import torch

for mb in (0.6, 1.6, 3.2, 64):
    n = int(mb * 2**20 / 4)
    src = torch.randn(n * 16).pin_memory()
    dst = torch.empty(n * 16, device="cuda")
    s = torch.cuda.Stream()
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with torch.cuda.stream(s):
            for it in range(200):
                i = it % 16
                dst[i * n:(i + 1) * n].copy_(src[i * n:(i + 1) * n], non_blocking=True)
        s.synchronize()
        el = time.perf_counter() - t
    print(f"chunk {mb:5.1f} MB: {200 * n * 4 / el / 1e9:6.1f} GB/s  ({el / 200 * 1e6:.1f} us/copy)", flush=True)
