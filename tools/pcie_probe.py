"""H2D bandwidth from pinned memory: one stream with large copies vs many streams with
small ones (the drop-in upload's pattern), alone and with a concurrent D2H."""
import time

import torch

dev = torch.device("cuda", 0)
N = 4 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device=dev)
hb = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
db = torch.empty(1 << 30, dtype=torch.uint8, device=dev)


def run(chunk, nstreams, d2h=False):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    k = 0
    for off in range(0, N, chunk):
        with torch.cuda.stream(streams[k % nstreams]):
            d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        k += 1
    if d2h:
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            for _ in range(1):
                hb.copy_(db, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return N / dt / 1e9


for chunk in (1 << 20, 3 << 19, 4 << 20, 64 << 20, 1 << 30):
    for ns in (1, 4, 15):
        run(chunk, ns)
        print(f"chunk {chunk >> 10:8d} KiB streams {ns:2d}: H2D {run(chunk, ns):6.1f} GB/s, with 1 GB D2H {run(chunk, ns, True):6.1f}",
              flush=True)
