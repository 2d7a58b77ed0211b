"""HBM write-only vs copy bandwidth on this GPU (context for the fp32-output tcgen05 epilogue):
torch fill_ (write-only) and copy_ (read + write) over 1 GiB, best of 10, CUDA events."""
import json

import torch


def best(fn, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    b = 1e9
    for _ in range(n):
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        b = min(b, e0.elapsed_time(e1))
    return b


a = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
c = torch.empty_like(a)
nb = a.numel() * 4
tw = best(lambda: a.fill_(1.0))
tc = best(lambda: c.copy_(a))
print(json.dumps({"write_only_gbs": nb / tw / 1e6, "copy_rw_gbs": 2 * nb / tc / 1e6, "bytes": nb}))
