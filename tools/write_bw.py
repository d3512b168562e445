"""Write-only and copy HBM bandwidth on this GPU (torch fill_ / copy_, CUDA events, best of 10):
the ceiling for write-dominated kernels such as the multi-plan payload pass (93% writes)."""
import json

import torch

n = 1 << 30  # 4 GiB of f32
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n, dtype=torch.float32, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def best(fn, bytes_):
    fn()
    torch.cuda.synchronize()
    out = 0.0
    for _ in range(10):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out = max(out, bytes_ / (s.elapsed_time(e) / 1e3) / 1e9)
    return round(out, 1)


print(json.dumps({"write_only_gbs": best(lambda: a.fill_(1.0), 4 * n),
                  "copy_gbs": best(lambda: b.copy_(a), 8 * n),
                  "how": "torch fill_ (write) and copy_ (read+write) over 4 GiB f32, best of 10"}))
