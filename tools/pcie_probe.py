import torch, time
dev = torch.device("cuda", 0)
N = 256 << 20  # 256 MiB
h = torch.empty(N, dtype=torch.uint8).pin_memory(); h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device=dev); d2 = torch.empty(N, dtype=torch.uint8, device=dev)
s = [torch.cuda.Stream() for _ in range(8)]
def run(kind, nstreams, chunk=16 << 20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for rep in range(4):
        for i, off in enumerate(range(0, N, chunk)):
            st = s[i % nstreams] if kind != "both" else None
            if kind == "h2d":
                with torch.cuda.stream(st): d[off:off+chunk].copy_(h[off:off+chunk], non_blocking=True)
            elif kind == "d2h":
                with torch.cuda.stream(st): h[off:off+chunk].copy_(d[off:off+chunk], non_blocking=True)
            else:
                with torch.cuda.stream(s[(i % nstreams)]): d[off:off+chunk].copy_(h[off:off+chunk], non_blocking=True)
                with torch.cuda.stream(s[4 + (i % nstreams)]): h2[off:off+chunk].copy_(d2[off:off+chunk], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    return 4 * N / dt / 1e9
for k in ("h2d", "d2h", "both"):
    for ns in (1, 2, 4):
        print(k, ns, "%.1f GB/s per direction" % run(k, ns))
for chunk_mb in (4, 8, 32):
    print("both", 2, f"chunk {chunk_mb} MiB", "%.1f GB/s per direction" % run("both", 2, chunk_mb << 20))
