#!/usr/bin/env python3
"""Microbenchmark: random int32 gathers from tables of various sizes
(L1/L2/HBM resident) -- the ceiling for the per-point cell-entry lookup."""
import json
import torch

N = 100_000_000
idx_src = torch.randint(0, 2**31 - 1, (N,), device="cuda", dtype=torch.int64)
for mb in (0.004, 1, 11, 42, 105, 400, 1600):
    n = max(1, int(mb * 1e6 / 4))
    table = torch.randint(0, 1000, (n,), device="cuda", dtype=torch.int32)
    idx = (idx_src % n).to(torch.int32)
    out = torch.empty(N, dtype=torch.int32, device="cuda")
    for _ in range(3):
        torch.index_select(table, 0, idx, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.index_select(table, 0, idx, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"table_MB": mb, "ms_per_100M": ms, "gathers_per_s": N / ms * 1e3}), flush=True)
# streaming copy reference: 16 B in + 4 B out per element
a = torch.empty((N, 2), dtype=torch.float64, device="cuda")
b = torch.empty(N, dtype=torch.int32, device="cuda")
for _ in range(3):
    b.copy_(a[:, 0])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    b.copy_(a[:, 0])
e1.record()
torch.cuda.synchronize()
print(json.dumps({"strided_copy_ms_per_100M": e0.elapsed_time(e1) / 10}))
