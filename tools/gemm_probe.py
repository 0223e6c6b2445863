"""Time the tcgen05 GEMM on the MoE layer's shapes (CUDA events, warm, L2 > working set
flushed between reps by a 256 MB write). Prints TFLOP/s per shape."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2411_16786_b200 import ops

dev = "cuda"
flush = torch.ones(64 * 2 ** 20, dtype=torch.float32, device=dev)  # 256 MB, read to evict L2


QUICK = "--quick" in __import__("sys").argv


def bench(M, N, K, epi, reps=20, label=""):
    A = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device=dev) * 0.05).to(torch.bfloat16)
    o16 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    o32 = torch.empty(M, N, device=dev) if epi in (2, 3, 4) else None
    res = torch.randn(M, N, device=dev) if epi in (3, 4) else None
    if epi == 4:   # shared GEMM2 + consume over two slots of pair rows
        rows = (torch.randn(2, M, N, device=dev) * 0.1).to(torch.bfloat16)
        gates = torch.rand(M, 2, device=dev)
        run = lambda: ops.gemm_consume(A, B, res, rows, gates, o32, o16)
    else:
        run = lambda: ops.gemm(epi, A, B, out_f32=o32, out_bf16=o16, residual=res)
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[len(ts) // 2] * 1e-3
    tf = 2.0 * M * N * K / t / 1e12
    if QUICK:
        print(f"{label:28s} M={M:6d} N={N:5d} K={K:5d} epi={epi}: {t*1e6:8.1f} us {tf:7.1f} TF/s",
              flush=True)
        return
    # torch reference time
    for _ in range(3):
        A @ B.T
    tt = []
    for _ in range(reps):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); A @ B.T; e1.record()
        torch.cuda.synchronize()
        tt.append(e0.elapsed_time(e1))
    tt.sort()
    ttf = 2.0 * M * N * K / (tt[len(tt) // 2] * 1e-3) / 1e12
    print(f"{label:28s} M={M:6d} N={N:5d} K={K:5d} epi={epi}: {t*1e6:8.1f} us {tf:7.1f} TF/s"
          f"   (cuBLAS plain {ttf:7.1f} TF/s)", flush=True)


if __name__ == "__main__":
    bench(8192, 1152, 1152, 3, label="local (gelu+resid)")
    bench(8192, 9216, 1152, 1, label="shared GEMM1 (gelu)")
    bench(8192, 1152, 9216, 4, label="shared GEMM2 (consume)")
    bench(16384, 4608, 1152, 1, label="expert GEMM1 (dense eq.)")
    bench(16384, 4608, 1152, 0, label="expert GEMM1 no-GELU")
    bench(16384, 1152, 4608, 0, label="expert GEMM2 (dense eq.)")
    if "--local" in __import__("sys").argv:
        for epi in (0, 2, 3):
            bench(8192, 1152, 1152, epi, label=f"local shape epi={epi}")
        for M in (2048, 4096, 16384, 32768):
            bench(M, 1152, 1152, 0, label=f"M={M} epi=0")
        bench(8192, 4608, 1152, 0, label="8192x4608x1152 epi=0")
        bench(8192, 1152, 2304, 0, label="8192x1152x2304 epi=0")
        raise SystemExit
    if "--consume" in __import__("sys").argv:
        for M in (8192, 9472):
            for epi in (0, 2, 4):
                bench(M, 1152, 9216, epi, label=f"consume shape M={M} epi={epi}")
        raise SystemExit
    if "--bn" in __import__("sys").argv:
        bench(16384, 4608, 4608, 0, label="16k x 4608 x 4608")
        bench(16384, 4608, 1152, 0, label="16k x 4608 x 1152")
        bench(16384, 1152, 4608, 0, label="16k x 1152 x 4608")
        bench(16384, 2304, 4608, 0, label="16k x 2304 x 4608")
        raise SystemExit
    if QUICK:
        raise SystemExit
    bench(8192, 8192, 8192, 0, label="square 8192")
    bench(9472, 1152, 9216, 4, label="GEMM2 consume, full waves")
    bench(18944, 1152, 4608, 0, label="GEMM2 expert, full waves")
