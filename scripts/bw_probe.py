"""HBM bandwidth of pure-write, copy (1:1) and 1:2 read:write streams on
this GPU (CUDA events, 8 GiB buffers), for the roofline of write-heavy
kernels (the lattice stencil writes 2 bytes per byte it reads)."""
import json
import torch

n = 1 << 30                       # 8 GiB of f64
a = torch.empty(n, dtype=torch.float64, device="cuda").fill_(1.0)
b = torch.empty_like(a)
c = torch.empty(n // 2, dtype=torch.float64, device="cuda")
res = {}


def timed(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e9
    for _ in range(reps):
        e[0].record()
        fn()
        e[1].record()
        torch.cuda.synchronize()
        best = min(best, e[0].elapsed_time(e[1]))
    return nbytes / (best * 1e-3) / 1e9


res["write_GBs"] = timed(lambda: b.fill_(2.0), 8 * n)
res["copy_1to1_GBs"] = timed(lambda: b.copy_(a), 16 * n)
# 1 : 2 -- read half of a, write it twice (into b's halves)
res["read1_write2_GBs"] = timed(lambda: torch.stack([a[:n // 2], a[:n // 2]], out=b.view(2, n // 2)),
                                8 * (n // 2) * 3)
res["read_GBs"] = timed(lambda: a.sum(), 8 * n)
print(json.dumps(res))
