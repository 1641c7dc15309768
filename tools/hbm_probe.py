"""HBM bandwidth of the three access mixes the codec kernels have: fill (write only, what encode is), copy (read + write,
what MEASURED_PEAKS.json quotes) and reduce (read only, what decode is).  torch kernels on a 4 GiB buffer, CUDA events."""
import json

import torch

n = 1 << 30                      # 4 GiB of int32
a = torch.empty(n, dtype=torch.int32, device="cuda")
b = torch.empty(n, dtype=torch.int32, device="cuda")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) * 1e-3 / reps


out = {}
t = timed(lambda: a.fill_(7))
out["fill_gbs"] = 4 * n / t / 1e9
t = timed(lambda: torch.cuda.current_stream().synchronize() or a.zero_())
out["memset_gbs"] = 4 * n / t / 1e9
t = timed(lambda: b.copy_(a))
out["copy_gbs"] = 8 * n / t / 1e9
t = timed(lambda: a.sum())
out["reduce_gbs"] = 4 * n / t / 1e9
t = timed(lambda: a.view(torch.int64).max())
out["reduce_max64_gbs"] = 4 * n / t / 1e9
print(json.dumps(out))
