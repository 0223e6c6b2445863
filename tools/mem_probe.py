"""Time the memory-bound MoE kernels at the bench shape (XL, 8192 rows, k=2, E=8)
with CUDA events and report achieved GB/s over their algorithmic bytes."""
import json
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_16786_b200 import ops

dev = "cuda"
n = int(sys.argv[sys.argv.index("--rows") + 1]) if "--rows" in sys.argv else 8192
k, E, h = 2, 8, 1152
hp = h
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6650.0
flush = torch.ones(64 * 2 ** 20, dtype=torch.float32, device=dev)  # 256 MB, read to evict L2


def timeit(fn, reps=20, batch=20):
    """Median over reps of (batch back-to-back launches)/batch, so host launch
    overhead overlaps device time; L2 evicted (read-flush) before each batch."""
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)   # keep the GPU busy while the batch is enqueued
        a.record()
        for _ in range(batch):
            fn()
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / batch)
    ts.sort()
    return ts[len(ts) // 2]


u32 = torch.randn(n, hp, device=dev)
u16 = u32.to(torch.bfloat16)
wg = torch.randn(E, hp, device=dev) * 0.03
ids = torch.empty(n, k, dtype=torch.int32, device=dev)
gates = torch.empty(n, k, device=dev)
us = timeit(lambda: ops.gate_topk(u32, wg, k, ids, gates))
byts = n * hp * 4 + E * hp * 4 + n * k * 8
print(f"gate_topk        {us:8.2f} us  {byts/us/1e3:8.1f} GB/s  ({byts/us/1e3/peak:.2f} of HBM)")

max_rows = ops.permute_max_rows(n, k, E)
x_perm = torch.empty(max_rows, hp, dtype=torch.bfloat16, device=dev)
pos = torch.empty(n, k, dtype=torch.int32, device=dev)
tiles = torch.empty(E + 1, dtype=torch.int32, device=dev)
cnt = torch.zeros(2, dtype=torch.int64, device=dev)
scr = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
us = timeit(lambda: ops.route_permute(ids, None, u16, x_perm, pos, tiles, cnt, scr, E))
byts = n * k * hp * 2 * 2 + n * k * 8
print(f"route_permute    {us:8.2f} us  {byts/us/1e3:8.1f} GB/s  ({byts/us/1e3/peak:.2f} of HBM)")

y = torch.randn(max_rows, hp, device=dev).to(torch.bfloat16)
routed = torch.empty(n, hp, device=dev)
us = timeit(lambda: ops.cache_assemble(y, pos, None, None, gates, ids, routed))
byts = n * k * hp * 2 + n * hp * 4 + n * k * 8
print(f"cache_assemble   {us:8.2f} us  {byts/us/1e3:8.1f} GB/s  ({byts/us/1e3/peak:.2f} of HBM)")

x16 = torch.empty(n, hp, dtype=torch.bfloat16, device=dev)
us = timeit(lambda: ops.denoise(u32, x16, routed, 1e-6))
byts = n * hp * (4 + 4 + 4 + 2)
print(f"denoise          {us:8.2f} us  {byts/us/1e3:8.1f} GB/s  ({byts/us/1e3/peak:.2f} of HBM)")
