"""One GEMM shape, three launches, for a single-kernel ncu capture of this
repo's tcgen05 GEMM or cuBLAS on the same operands:

  ncu --set full -k regex:'gemm_bf16_pair|nvjet' -s 2 -c 1 -o OUT \\
      python tools/gemm_one.py M N K EPI {ours|cublas}
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2411_16786_b200 import ops  # noqa: E402

M, N, K, epi = (int(v) for v in sys.argv[1:5])
impl = sys.argv[5]
dev = "cuda"
A = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
B = (torch.randn(N, K, device=dev) * 0.05).to(torch.bfloat16)
o16 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
o32 = torch.empty(M, N, device=dev) if epi in (2, 3, 4) else None
res = torch.randn(M, N, device=dev) if epi in (3, 4) else None
for _ in range(3):
    if impl == "cublas":
        A @ B.T
    elif epi == 4:
        rows = torch.zeros(2, M, N, device=dev, dtype=torch.bfloat16)
        ops.gemm_consume(A, B, res, rows, torch.zeros(M, 2, device=dev), o32, o16)
    else:
        ops.gemm(epi, A, B, out_f32=o32, out_bf16=o16, residual=res)
torch.cuda.synchronize()
