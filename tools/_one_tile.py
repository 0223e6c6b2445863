import sys, torch
sys.path.insert(0, ".")
from paper_2411_16786_b200 import ops
A = (torch.randn(256, 1152, device="cuda") * 0.5).to(torch.bfloat16)
B = (torch.randn(1152, 1152, device="cuda") * 0.05).to(torch.bfloat16)
o16 = torch.empty(256, 1152, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    ops.gemm(0, A, B, out_bf16=o16)
torch.cuda.synchronize()
