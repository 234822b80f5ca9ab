import torch, time
n = 16 * (1 << 20) // 4
for streams in (1, 4, 16):
    src = [torch.randn(n).pin_memory() for _ in range(8)]
    dst = [torch.empty(n, device="cuda") for _ in range(8)]
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    for rep in range(2):
        t = time.perf_counter()
        for it in range(64):
            with torch.cuda.stream(ss[it % streams]):
                dst[it % 8].copy_(src[it % 8], non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t
    print(f"streams={streams} 16MB copies: {64 * n * 4 / el / 1e9:.1f} GB/s")
# 1 MB chunks
m = (1 << 20) // 4
src = torch.randn(m * 64).pin_memory(); dst = torch.empty(m * 64, device="cuda")
ss = [torch.cuda.Stream() for _ in range(16)]
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    for it in range(2048):
        i = it % 64
        with torch.cuda.stream(ss[it % 16]):
            dst[i*m:(i+1)*m].copy_(src[i*m:(i+1)*m], non_blocking=True)
    torch.cuda.synchronize(); el = time.perf_counter() - t
print(f"1MB copies x16 streams: {2048 * m * 4 / el / 1e9:.1f} GB/s")
