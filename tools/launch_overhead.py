"""Per-launch cost of the tcgen05 GEMM inside a CUDA graph: 20 back-to-back
identical launches captured once, replayed, time per launch. Small M isolates
the fixed cost (prologue: barrier init, TMEM alloc, cluster sync, pipeline
fill; epilogue drain) from the per-tile cost."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_16786_b200 import ops

dev = "cuda"


def per_launch(M, N, K, epi, reps=20):
    A = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device=dev) * 0.05).to(torch.bfloat16)
    o16 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    o32 = torch.empty(M, N, device=dev) if epi in (2, 3, 4) else None
    res = torch.randn(M, N, device=dev) if epi in (3, 4) else None
    run = lambda: ops.gemm(epi, A, B, out_f32=o32, out_bf16=o16, residual=res)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            run()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
    print(f"M={M:6d} N={N:5d} K={K:5d} epi={epi}: {us:7.2f} us/launch  {2*M*N*K/us/1e6:7.1f} TF/s", flush=True)


for M in (256, 2048, 8192):
    per_launch(M, 1152, 1152, 0)
per_launch(8192, 1152, 1152, 3)
per_launch(8192, 9216, 1152, 1)
