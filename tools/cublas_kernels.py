"""Which cuBLAS kernels (tile shape, cluster shape, grid) serve the MoE layer's
GEMM shapes on this GPU: run under ncu's LaunchStats section, e.g.

  ncu --section LaunchStats --csv --log-file gpurun_out/cublas.csv python tools/cublas_kernels.py

(the kernel names encode cuBLAS's tile / cluster choice; the comparison point
for the tcgen05 GEMM's tiling)."""
import torch

dev = "cuda"
SHAPES = [  # (M, N, K, label)
    (8192, 1152, 9216, "shared GEMM2 (consume)"),
    (8192, 1152, 1152, "local"),
    (16384, 4608, 1152, "expert GEMM1"),
    (16384, 1152, 4608, "expert GEMM2"),
]
for M, N, K, label in SHAPES:
    A = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device=dev) * 0.05).to(torch.bfloat16)
    for _ in range(2):
        A @ B.T
    torch.cuda.synchronize()
    print(label, M, N, K, flush=True)
