"""HBM ceilings by access mix on this box (context for the f2 scores, which only
write): copy (read+write), write-only (fill), read-only (sum) over 4 GiB, CUDA events,
best of 10.  Not a bench value; prints one JSON line."""
import json
import torch

n = 1 << 31                      # bf16 elements: 4 GiB
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
a.normal_()


def best(fn, nbytes, reps=10):
    t = []
    for _ in range(reps + 2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        t.append(s.elapsed_time(e))
    return nbytes / (min(t[2:]) * 1e-3) / 1e9


out = {
    "copy_gbs": best(lambda: b.copy_(a), 4 * n),
    "fill_gbs": best(lambda: b.fill_(1.0), 2 * n),
    "zero_gbs": best(lambda: b.zero_(), 2 * n),
    "read_sum_gbs": best(lambda: a.view(torch.int32).sum(dtype=torch.int64), 2 * n),
}
print(json.dumps({k: round(v, 1) for k, v in out.items()}))
