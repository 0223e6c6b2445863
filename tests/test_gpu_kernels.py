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


@pytest.mark.parametrize("M,E,k", [(8192, 8, 2), (1000, 8, 2), (777, 16, 2), (256, 8, 3), (130, 16, 5)])
def test_local_gemm_fused_gate(M, E, k):
    """local_block GEMM with the router's partial logits fused into its epilogue
    + the finish kernel vs the unfused GELU_RESID GEMM + dice_gate_topk: u
    bit-identical, ids identical outside the tie band, gates/scores within fp32
    reassociation (the logit sum order differs), decide masks identical."""
    hp = 1152
    g = torch.Generator(device=dev).manual_seed(M + E + k)
    x32 = torch.randn(M, hp, device=dev, generator=g)
    x16 = x32.to(torch.bfloat16)
    W = (torch.randn(hp, hp, device=dev, generator=g) / np.sqrt(hp)).to(torch.bfloat16)
    wg_t = (torch.rand(E, hp, device=dev, generator=g) * 2 - 1) / np.sqrt(hp)
    wg_c = wg_t.t().contiguous()
    u32a = torch.empty(M, hp, device=dev); u16a = torch.empty(M, hp, device=dev, dtype=torch.bfloat16)
    u32b = torch.empty_like(u32a); u16b = torch.empty_like(u16a)
    ops.gemm(ops.EPI_GELU_RESID, x16, W, out_f32=u32a, out_bf16=u16a, residual=x32)
    P = ops.gate_parts(M, hp, hp, E)
    parts = torch.empty(P, M, E, device=dev)
    ops.gemm_local_gate(x16, W, wg_c, u32b, u16b, x32, parts)
    assert torch.equal(u32a, u32b) and torch.equal(u16a, u16b)
    ids_a = torch.empty(M, k, dtype=torch.int32, device=dev); gates_a = torch.empty(M, k, device=dev)
    sc_a = torch.empty(M, E, device=dev)
    ids_b = torch.empty_like(ids_a); gates_b = torch.empty_like(gates_a); sc_b = torch.empty_like(sc_a)
    st = torch.empty(4, dtype=torch.int32, device=dev)
    ops.status_reset(st)
    ops.gate_topk(u32a, wg_t, k, ids_a, gates_a, sc_a, st, 0, 0)
    # logits in fp64 from the same u, for the tie band
    logits = u32a.double() @ wg_c.double()
    sc = torch.softmax(logits, dim=1)
    top = torch.sort(sc, dim=1, descending=True).values
    gap = (top[:, :k] - top[:, 1:k + 1]).abs().min(dim=1).values
    clear = gap > 1e-5
    # fused finish, with the cond decision fused (LowScore, R=2, step 0: all due)
    n = M
    last = torch.full((n,), -10 ** 9, dtype=torch.int32, device=dev)
    primed = torch.zeros(n, dtype=torch.uint8, device=dev)
    red = torch.zeros(n, k, dtype=torch.uint8, device=dev)
    cids = torch.full((n, k), -1, dtype=torch.int32, device=dev)
    act_b = torch.empty(n, k, dtype=torch.uint8, device=dev); wr_b = torch.empty_like(act_b)
    dec = (False, 2, ops.COND_CODES["low_score"], False, 0, last, primed, red, cids, act_b, wr_b)
    ops.gate_finish(parts, ids_b, gates_b, sc_b, st, 0, 0, decide=dec)
    torch.cuda.synchronize()
    assert int(st[0].item()) == 2 ** 31 - 1
    assert torch.equal(ids_a[clear], ids_b[clear])
    assert (gates_a - gates_b).abs().max().item() < 1e-5
    assert (sc_a - sc_b).abs().max().item() < 1e-5
    # same decision as the standalone kernel on the fused ids
    last2 = torch.full((n,), -10 ** 9, dtype=torch.int32, device=dev)
    primed2 = torch.zeros(n, dtype=torch.uint8, device=dev)
    red2 = torch.zeros(n, k, dtype=torch.uint8, device=dev)
    act_a = torch.empty_like(act_b); wr_a = torch.empty_like(wr_b)
    ops.cond_decide(ids_b, 0, False, 2, "low_score", False, 0, last2, primed2, red2, cids, act_a, wr_a)
    torch.cuda.synchronize()
    for a_, b_ in ((act_a, act_b), (wr_a, wr_b), (last2, last), (primed2, primed), (red2, red)):
        assert torch.equal(a_, b_)


def test_fused_gate_nonfinite_flag():
    M, hp, E = 300, 1152, 8
    x32 = torch.zeros(M, hp, device=dev)
    x32[123, 7] = float("inf")
    W = torch.zeros(hp, hp, device=dev, dtype=torch.bfloat16)
    wg_c = torch.ones(hp, E, device=dev) * 1e-3
    u32 = torch.empty(M, hp, device=dev); u16 = torch.empty(M, hp, device=dev, dtype=torch.bfloat16)
    parts = torch.empty(ops.gate_parts(M, hp, hp, E), M, E, device=dev)
    ops.gemm_local_gate(x32.to(torch.bfloat16), W, wg_c, u32, u16, x32, parts)
    ids = torch.empty(M, 2, dtype=torch.int32, device=dev); gates = torch.empty(M, 2, device=dev)
    st = torch.empty(4, dtype=torch.int32, device=dev)
    ops.status_reset(st)
    ops.gate_finish(parts, ids, gates, None, st, 5, 3)
    torch.cuda.synchronize()
    assert st[:2].tolist() == [5, 3]


@pytest.mark.parametrize("n,E,k,hp,strategy,strict", [(8192, 8, 2, 1152, "low_score", False),
                                                      (999, 16, 2, 640, "random", True),
                                                      (300, 8, 3, 128, "high_score", False),
                                                      (77, 4, 2, 64, "low_score", True)])
def test_gate_topk_with_fused_decide(n, E, k, hp, strategy, strict):
    """dice_gate_topk_decide == dice_gate_topk then dice_cond_decide (same
    kernel for the gate, so ids/gates are bit-identical), over a few steps of
    evolving cache state."""
    g = torch.Generator(device=dev).manual_seed(n + E)
    wg = (torch.rand(E, hp, device=dev, generator=g) * 2 - 1) / np.sqrt(hp)
    st = {}
    for name in ("a", "b"):
        st[name] = dict(last=torch.full((n,), -10 ** 9, dtype=torch.int32, device=dev),
                        primed=torch.zeros(n, dtype=torch.uint8, device=dev),
                        red=torch.zeros(n, k, dtype=torch.uint8, device=dev),
                        cids=torch.randint(0, E, (n, k), dtype=torch.int32, device=dev, generator=g))
    st["b"]["cids"] = st["a"]["cids"].clone()
    status = torch.empty(4, dtype=torch.int32, device=dev)
    ops.status_reset(status)
    for step in range(5):
        u = torch.randn(n, hp, device=dev, generator=g)
        out = {}
        for name in ("a", "b"):
            s_ = st[name]
            ids = torch.empty(n, k, dtype=torch.int32, device=dev)
            gates = torch.empty(n, k, device=dev)
            act = torch.empty(n, k, dtype=torch.uint8, device=dev)
            wr = torch.empty_like(act)
            force = step == 3
            if name == "a":
                ops.gate_topk(u, wg, k, ids, gates, None, status, step, 0)
                ops.cond_decide(ids, step, force, 2, strategy, strict, 0x1234 + step, s_["last"],
                                s_["primed"], s_["red"], s_["cids"], act, wr)
            else:
                dec = (force, 2, ops.COND_CODES[strategy], strict, 0x1234 + step, s_["last"],
                       s_["primed"], s_["red"], s_["cids"], act, wr)
                ops.gate_topk(u, wg, k, ids, gates, None, status, step, 0, decide=dec)
            out[name] = (ids, gates, act, wr)
        for x, y in zip(out["a"], out["b"]):
            assert torch.equal(x, y)
        for key in ("last", "primed", "red"):
            assert torch.equal(st["a"][key], st["b"][key])


@pytest.mark.parametrize("n,k,E,devices,masked", [(8192, 2, 8, 1, True), (8192, 2, 8, 4, False),
                                                  (1000, 3, 16, 2, True), (37, 2, 8, 1, False),
                                                  (32768, 2, 16, 8, True)])
@pytest.mark.parametrize("fused", ["0", "1"])
def test_route_permute_single_launch(n, k, E, devices, masked, fused, monkeypatch):
    """The single-launch permute (count -> grid barrier -> positions -> grid
    barrier -> gather) against a numpy restatement of the grouping: pairs of
    an expert in pair order t*k+s, experts padded to 256-row tiles, inactive
    pairs -1, byte-plan counters (cluster.py:75-90); repeated launches reuse
    the barrier state. Both the three-kernel path and the single launch
    (DICE_PERMUTE_FUSED=1, read per call) are checked."""
    monkeypatch.setenv("DICE_PERMUTE_FUSED", fused)
    hp = 128
    g = torch.Generator(device=dev).manual_seed(n + k + E)
    ids = torch.randint(0, E, (n, k), dtype=torch.int32, device=dev, generator=g)
    active = (torch.rand(n, k, device=dev, generator=g) > 0.3).to(torch.uint8) if masked else None
    u16 = torch.randn(n, hp, device=dev, generator=g).to(torch.bfloat16)
    max_rows = ops.permute_max_rows(n, k, E)
    scratch = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
    idn = ids.cpu().numpy().reshape(-1)
    act = np.ones(n * k, bool) if active is None else active.cpu().numpy().reshape(-1).astype(bool)
    pos_ref = np.full(n * k, -1, np.int64)
    tiles, base = [0], 0
    for e in range(E):
        sel = np.nonzero((idn == e) & act)[0]
        pos_ref[sel] = base + np.arange(len(sel))
        nt = (len(sel) + 255) // 256
        base += nt * 256
        tiles.append(tiles[-1] + nt)
    homes = (np.arange(n) * devices) // n
    t_of = np.arange(n * k) // k
    remote = act & (homes[t_of] != idn // (E // devices))
    for rep in range(3):
        x_perm = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
        pos = torch.empty(n, k, dtype=torch.int32, device=dev)
        tile_off = torch.empty(E + 1, dtype=torch.int32, device=dev)
        counters = torch.zeros(2, dtype=torch.int64, device=dev)
        ops.route_permute(ids, active, u16, x_perm, pos, tile_off, counters, scratch, E,
                          devices=devices, row0=0, rows_total=n)
        torch.cuda.synchronize()
        assert np.array_equal(pos.cpu().numpy().reshape(-1), pos_ref)
        assert tile_off.cpu().tolist() == tiles
        assert counters.cpu().tolist() == [int(act.sum()), int(remote.sum())]
        v = pos_ref >= 0
        assert torch.equal(x_perm[torch.as_tensor(pos_ref[v], device=dev)],
                           u16[torch.as_tensor(t_of[v], device=dev)])


def test_expert_gemm1_with_shared_dual_launch():
    """Grouped expert GEMM1 + the dense shared GEMM1 in one persistent launch:
    bit-identical to the two separate launches (same tiles, same epilogue)."""
    n, k, E, hp, ep, S = 3000, 2, 8, 1152, 512, 2
    g = torch.Generator(device=dev).manual_seed(11)
    ids = torch.randint(0, E, (n, k), dtype=torch.int32, device=dev, generator=g)
    u16 = (torch.randn(n, hp, device=dev, generator=g) * 0.5).to(torch.bfloat16)
    w1 = (torch.randn(E * ep, hp, device=dev, generator=g) / 34).to(torch.bfloat16)
    w2 = (torch.randn(E * hp, ep, device=dev, generator=g) / 23).to(torch.bfloat16)
    ws1 = (torch.randn(S * ep, hp, device=dev, generator=g) / 34).to(torch.bfloat16)
    max_rows = ops.permute_max_rows(n, k, E)
    x_perm = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
    pos = torch.empty(n, k, dtype=torch.int32, device=dev)
    tiles = torch.empty(E + 1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    scr = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
    ops.route_permute(ids, None, u16, x_perm, pos, tiles, cnt, scr, E)
    h_a = torch.zeros(max_rows, ep, dtype=torch.bfloat16, device=dev)
    y_a = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
    hs_a = torch.zeros(n, S * ep, dtype=torch.bfloat16, device=dev)
    ops.grouped_ffn(x_perm, w1, w2, E, tiles, h_a, y_a)
    ops.gemm(ops.EPI_GELU_BF16, u16, ws1, out_bf16=hs_a)
    h_b, y_b, hs_b = torch.zeros_like(h_a), torch.zeros_like(y_a), torch.zeros_like(hs_a)
    ops.expert_gemm1_with_shared(x_perm, w1, E, tiles, h_b, u16, ws1, hs_b)
    ops.expert_gemm2(h_b, w2, E, tiles, y_b)
    torch.cuda.synchronize()
    nt = int(tiles[-1].item()) * 256
    assert torch.equal(h_a[:nt], h_b[:nt]) and torch.equal(y_a[:nt], y_b[:nt])
    assert torch.equal(hs_a, hs_b)


@pytest.mark.parametrize("k,masked", [(2, True), (2, False), (1, True)])
def test_fused_combine_matches_cache_assemble(k, masked):
    """Routed combine in the expert GEMM2 epilogue (slot init with the cached
    terms + float4 atomic adds of round(g * row)) == expert GEMM2 then
    cache_assemble: combine slot, cache rows, gates and ids bit-identical, and
    run-to-run identical (k <= 2 terms per token commute)."""
    n, E, hp, ep = 2000, 8, 1152, 512
    g = torch.Generator(device=dev).manual_seed(21 + k)
    ids = torch.randint(0, E, (n, k), dtype=torch.int32, device=dev, generator=g)
    gates = torch.rand(n, k, device=dev, generator=g)
    u16 = (torch.randn(n, hp, device=dev, generator=g) * 0.5).to(torch.bfloat16)
    w1 = (torch.randn(E * ep, hp, device=dev, generator=g) / 34).to(torch.bfloat16)
    w2 = (torch.randn(E * hp, ep, device=dev, generator=g) / 23).to(torch.bfloat16)
    if masked:
        active = (torch.rand(n, k, device=dev, generator=g) > 0.35).to(torch.uint8)
        write = ((torch.rand(n, k, device=dev, generator=g) > 0.5).to(torch.uint8) * active)
    else:
        active = write = None
    rows0 = (torch.randn(k, n, hp, device=dev, generator=g)).to(torch.bfloat16)
    cg0 = torch.rand(n, k, device=dev, generator=g)
    ci0 = torch.randint(0, E, (n, k), dtype=torch.int32, device=dev, generator=g)
    max_rows = ops.permute_max_rows(n, k, E)
    x_perm = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
    pos = torch.empty(n, k, dtype=torch.int32, device=dev)
    tiles = torch.empty(E + 1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    scr = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
    row_pair = torch.empty(max_rows, dtype=torch.int32, device=dev)
    ops.route_permute(ids, active, u16, x_perm, pos, tiles, cnt, scr, E, row_pair=row_pair)
    hbuf = torch.zeros(max_rows, ep, dtype=torch.bfloat16, device=dev)
    y = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
    # reference path
    rows_a, cg_a, ci_a = rows0.clone(), cg0.clone(), ci0.clone()
    slot_a = torch.full((n, hp), float("nan"), device=dev)
    ops.grouped_ffn(x_perm, w1, w2, E, tiles, hbuf, y)
    ops.cache_assemble(y, pos, active, write, gates, ids, slot_a, rows_a if masked else None,
                       cg_a if masked else None, ci_a if masked else None)
    outs = []
    for _ in range(2):
        rows_b, cg_b, ci_b = rows0.clone(), cg0.clone(), ci0.clone()
        slot_b = torch.full((n, hp), float("nan"), device=dev)
        ops.slot_init(active, write, gates, ids, slot_b, rows_b if masked else None,
                      cg_b if masked else None, ci_b if masked else None)
        ops.expert_gemm2_combine(hbuf, w2, E, tiles, row_pair, gates, write, slot_b,
                                 rows_b if masked else None)
        torch.cuda.synchronize()
        outs.append(slot_b.clone())
        assert torch.equal(slot_b, slot_a)
        if masked:
            assert torch.equal(rows_b, rows_a) and torch.equal(cg_b, cg_a) and torch.equal(ci_b, ci_a)
    assert torch.equal(outs[0], outs[1])


def test_gemm_rejects_internal_epilogue_kinds():
    A = torch.zeros(256, 64, device=dev, dtype=torch.bfloat16)
    B = torch.zeros(64, 64, device=dev, dtype=torch.bfloat16)
    o = torch.empty(256, 64, device=dev, dtype=torch.bfloat16)
    from paper_2411_16786_b200.errors import ContractError
    for epi in (-1, 5, 6, 7, 99):
        with pytest.raises(ContractError):
            ops.gemm(epi, A, B, out_bf16=o)


@pytest.mark.parametrize("n,k,devices", [(8192, 2, 2), (1000, 2, 1), (777, 1, 4), (300, 4, 8)])
def test_gate_counted_permute_matches_count_kernel(n, k, devices):
    """dice_gate_topk_counted + dice_route_permute_counted == dice_gate_topk +
    dice_route_permute: ids, gates, positions, tile offsets, permuted rows and
    the run counters (active / remote pairs under D simulated devices). (The
    engine test covers the decide-masked path.)"""
    E, hp = 8, 256
    g = torch.Generator(device=dev).manual_seed(n + k)
    u = torch.randn(n, hp, device=dev, generator=g)
    wg = torch.randn(E, hp, device=dev, generator=g) * 0.1
    u16 = u.to(torch.bfloat16)
    max_rows = ops.permute_max_rows(n, k, E)
    res = {}
    for mode in ("count", "plain"):
        ids = torch.empty(n, k, dtype=torch.int32, device=dev)
        gates = torch.empty(n, k, device=dev)
        cnt = torch.zeros(2, dtype=torch.int64, device=dev)
        pos = torch.empty(n, k, dtype=torch.int32, device=dev)
        tiles = torch.empty(E + 1, dtype=torch.int32, device=dev)
        x_perm = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
        if mode == "count":
            cc = torch.zeros((n + 31) // 32 * 8, dtype=torch.int32, device=dev)
            ops.gate_topk(u, wg, k, ids, gates, count=(cc, cnt, devices, n))
            ops.route_permute(ids, None, u16, x_perm, pos, tiles, cnt, None, E, chunk_counts=cc)
        else:
            scr = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
            ops.gate_topk(u, wg, k, ids, gates)
            ops.route_permute(ids, None, u16, x_perm, pos, tiles, cnt, scr, E, devices=devices,
                              rows_total=n)
        torch.cuda.synchronize()
        res[mode] = (ids, gates, pos, tiles, x_perm, cnt)
    for a, b in zip(res["count"], res["plain"]):
        assert torch.equal(a, b)
