"""Kernel-level parity on the GPU: tcgen05 GEMM vs a torch fp32 reference of
the same bf16 operands; splitmix fill bit-exact vs the oracle stream."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import dice_oracle as O  # noqa: E402
from paper_2411_16786_b200 import ops  # noqa: E402

dev = "cuda"


def gelu(x):
    return 0.5 * x * (1.0 + torch.erf(x / np.sqrt(2.0)))


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 128, 128), (1000, 192, 1152),
                                   (64, 64, 64), (513, 1152, 640), (2048, 4608, 1152),
                                   (4096, 1152, 4608), (300, 768, 256), (777, 384, 128)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3, 4])
def test_dense_gemm_epilogues(M, N, K, epi):
    g = torch.Generator(device=dev).manual_seed(M * 7 + N + K + epi)
    A = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device=dev, generator=g) / np.sqrt(K)).to(torch.bfloat16)
    acc = A.float() @ B.float().T
    res = torch.randn(M, N, device=dev, generator=g)
    add = torch.randn(M, N, device=dev, generator=g)
    o32 = torch.full((M, N), float("nan"), device=dev)
    o16 = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    kw = {}
    if epi == 0:
        ref = acc; kw = dict(out_bf16=o16)
    elif epi == 1:
        ref = gelu(acc); kw = dict(out_bf16=o16)
    elif epi == 2:
        ref = acc; kw = dict(out_f32=o32, out_bf16=o16)
    elif epi == 3:
        ref = gelu(acc) + res; kw = dict(out_f32=o32, out_bf16=o16, residual=res)
    else:
        ref = res + (acc + add); kw = dict(out_f32=o32, out_bf16=o16, residual=res, addend=add)
    ops.gemm(epi, A, B, **kw)
    torch.cuda.synchronize()
    scale = ref.abs().max().item() + 1e-6
    if "out_f32" in kw:
        err = (o32 - ref).abs().max().item() / scale
        assert err < 1e-4, err
    err16 = (o16.float() - ref).abs().max().item() / scale
    assert err16 < 1e-2, err16


def test_splitmix_fill_bit_exact_f64():
    seed, start, rows, cols = 0xDEADBEEF, 12345, 37, 53
    out = torch.empty(rows, cols, dtype=torch.float64, device=dev)
    ops.splitmix_fill(out, seed, start, rows, cols, 0.125)
    ref = O.to_uniform(O.stream_bits(seed, start, rows * cols), 0.125).reshape(rows, cols)
    assert np.array_equal(out.cpu().numpy(), ref)
    outT = torch.empty(cols, rows, dtype=torch.float64, device=dev)
    ops.splitmix_fill(outT, seed, start, rows, cols, 0.125, transpose=True)
    assert np.array_equal(outT.cpu().numpy(), ref.T)
    o32 = torch.empty(rows, cols, dtype=torch.float32, device=dev)
    ops.splitmix_fill(o32, seed, start, rows, cols, 0.125)
    assert np.array_equal(o32.cpu().numpy(), ref.astype(np.float32))
    bits = ops.splitmix_bits(seed, start, 100).cpu().numpy().view(np.uint64)
    assert np.array_equal(bits, O.stream_bits(seed, start, 100))


def test_stream_k_path_matches_data_parallel():
    """The opt-in stream-K schedule (DICE_GEMM_STREAMK=1, read once per process)
    must give the same GEMM results; run in a subprocess with the variable set."""
    import subprocess, sys, os
    code = r"""
import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2411_16786_b200 import ops
g = torch.Generator(device='cuda').manual_seed(0)
for (M, N, K, epi) in [(8192, 1152, 1152, 3), (2048, 1152, 4608, 0), (4096, 1152, 2304, 4)]:
    A = torch.randn(M, K, device='cuda', generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device='cuda', generator=g) / K ** 0.5).to(torch.bfloat16)
    res = torch.randn(M, N, device='cuda', generator=g)
    add = torch.randn(M, N, device='cuda', generator=g)
    o32 = torch.empty(M, N, device='cuda')
    kw = dict(out_f32=o32)
    acc = A.float() @ B.float().T
    if epi == 3:
        ref = 0.5 * acc * (1 + torch.erf(acc / 2 ** 0.5)) + res; kw['residual'] = res
    elif epi == 4:
        ref = res + (acc + add); kw.update(residual=res, addend=add)
    else:
        ref = acc; epi = 2
    ops.gemm(epi, A, B, **kw)
    torch.cuda.synchronize()
    err = ((o32 - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-4, (M, N, K, err)
print('ok')
"""
    env = dict(os.environ, DICE_GEMM_STREAMK="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
