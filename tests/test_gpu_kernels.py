"""Kernel-level parity on the GPU: tcgen05 GEMM vs a torch fp32 reference of
the same bf16 operands; splitmix fill bit-exact vs the oracle stream."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import dice_oracle as O  # noqa: E402
from paper_2411_16786_b200 import ops  # noqa: E402
import paper_2411_16786_b200 as D  # noqa: E402

dev = "cuda"


def gelu(x):
    return 0.5 * x * (1.0 + torch.erf(x / np.sqrt(2.0)))


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 128, 128), (1000, 192, 1152),
                                   (64, 64, 64), (513, 1152, 640), (2048, 4608, 1152),
                                   (4096, 1152, 4608), (300, 768, 256), (777, 384, 128)])
@pytest.mark.parametrize("epi", [0, 1, 2, 3])
def test_dense_gemm_epilogues(M, N, K, epi):
    g = torch.Generator(device=dev).manual_seed(M * 7 + N + K + epi)
    A = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device=dev, generator=g) / np.sqrt(K)).to(torch.bfloat16)
    acc = A.float() @ B.float().T
    res = torch.randn(M, N, device=dev, generator=g)
    o32 = torch.full((M, N), float("nan"), device=dev)
    o16 = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    kw = {}
    if epi == 0:
        ref = acc; kw = dict(out_bf16=o16)
    elif epi == 1:
        ref = gelu(acc); kw = dict(out_bf16=o16)
    elif epi == 2:
        ref = acc; kw = dict(out_f32=o32, out_bf16=o16)
    else:
        ref = gelu(acc) + res; kw = dict(out_f32=o32, out_bf16=o16, residual=res)
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
def test_route_permute_grouping(n, k, E, devices, masked):
    """The permute (count -> positions -> gather) against a numpy restatement
    of the grouping: pairs of an expert in pair order t*k+s, experts padded to
    256-row tiles, inactive pairs -1, the row -> pair map (-1 on padding rows),
    byte-plan counters (cluster.py:75-90); repeated launches give the same."""
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
    row_pair_ref = np.full(max_rows, -1, np.int64)
    row_pair_ref[pos_ref[pos_ref >= 0]] = np.nonzero(pos_ref >= 0)[0]
    for rep in range(3):
        x_perm = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
        pos = torch.empty(n, k, dtype=torch.int32, device=dev)
        tile_off = torch.empty(E + 1, dtype=torch.int32, device=dev)
        counters = torch.zeros(2, dtype=torch.int64, device=dev)
        row_pair = torch.full((max_rows,), 12345, dtype=torch.int32, device=dev)
        ops.route_permute(ids, active, u16, x_perm, pos, tile_off, counters, scratch, E,
                          devices=devices, row0=0, rows_total=n, row_pair=row_pair)
        torch.cuda.synchronize()
        assert np.array_equal(pos.cpu().numpy().reshape(-1), pos_ref)
        nt = tiles[-1] * 256
        assert np.array_equal(row_pair.cpu().numpy()[:nt], row_pair_ref[:nt])
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


@pytest.mark.parametrize("k,masked,E", [(2, True, 8), (2, False, 8), (1, True, 8), (3, True, 16)])
def test_expert_gemm2_pair_rows(k, masked, E):
    """Expert GEMM2 with the pair-row store epilogue == expert GEMM2 into y then
    a scatter: every active pair's bf16 row lands at pair_rows[s, t] and its
    gate / id in the cache arrays; inactive pairs keep their previous (cached)
    entries bit for bit; padding rows write nothing."""
    n, hp, ep = 2000, 1152, 512
    g = torch.Generator(device=dev).manual_seed(21 + k + E)
    ids = torch.randint(0, E, (n, k), dtype=torch.int32, device=dev, generator=g)
    gates = torch.rand(n, k, device=dev, generator=g)
    u16 = (torch.randn(n, hp, device=dev, generator=g) * 0.5).to(torch.bfloat16)
    w1 = (torch.randn(E * ep, hp, device=dev, generator=g) / 34).to(torch.bfloat16)
    w2 = (torch.randn(E * hp, ep, device=dev, generator=g) / 23).to(torch.bfloat16)
    active = ((torch.rand(n, k, device=dev, generator=g) > 0.35).to(torch.uint8)
              if masked else None)
    rows0 = torch.randn(k, n, hp, device=dev, generator=g).to(torch.bfloat16)
    cg0 = torch.rand(n, k, device=dev, generator=g)
    ci0 = torch.randint(0, E, (n, k), dtype=torch.int32, device=dev, generator=g)
    max_rows = ops.permute_max_rows(n, k, E)
    x_perm = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
    pos = torch.empty(n, k, dtype=torch.int32, device=dev)
    tiles = torch.empty(E + 1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    scr = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
    row_pair = torch.full((max_rows,), -1, dtype=torch.int32, device=dev)
    ops.route_permute(ids, active, u16, x_perm, pos, tiles, cnt, scr, E, row_pair=row_pair)
    hbuf = torch.zeros(max_rows, ep, dtype=torch.bfloat16, device=dev)
    y = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
    ops.grouped_ffn(x_perm, w1, w2, E, tiles, hbuf, y)
    # reference: y rows scattered to their pairs
    act = torch.ones(n, k, dtype=torch.bool, device=dev) if active is None else active.bool()
    rows_ref, cg_ref, ci_ref = rows0.clone(), cg0.clone(), ci0.clone()
    tt, ss = torch.nonzero(act, as_tuple=True)
    rows_ref[ss, tt] = y[pos[tt, ss].long()]
    cg_ref[act] = gates[act]
    ci_ref[act] = ids[act]
    for _ in range(2):
        rows, cg, ci = rows0.clone(), cg0.clone(), ci0.clone()
        ops.expert_gemm2_pairs(hbuf, w2, E, tiles, row_pair, gates, ids, rows, cg, ci)
        torch.cuda.synchronize()
        assert torch.equal(rows, rows_ref)
        assert torch.equal(cg, cg_ref) and torch.equal(ci, ci_ref)


@pytest.mark.parametrize("M,K,k", [(8192, 9216, 2), (1000, 512, 2), (777, 640, 1), (300, 256, 3)])
def test_gemm_consume(M, K, k):
    """Shared GEMM2 with the consume epilogue vs torch fp32 of the same bf16
    operands: out = u + ((acc + g_0 row_0) + g_1 row_1 ...) (schedules.py:317,
    model.py:295-297), and the S = 0 consume kernel vs the same formula."""
    N = 1152
    g = torch.Generator(device=dev).manual_seed(M + K + k)
    A = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device=dev, generator=g) / np.sqrt(K)).to(torch.bfloat16)
    u = torch.randn(M, N, device=dev, generator=g)
    rows = torch.randn(k, M, N, device=dev, generator=g).to(torch.bfloat16)
    gates = torch.rand(M, k, device=dev, generator=g)
    acc = A.float() @ B.float().T
    ref = acc.clone()
    for s in range(k):
        ref = ref + gates[:, s:s + 1] * rows[s].float()
    ref = u + ref
    o32 = torch.full((M, N), float("nan"), device=dev)
    o16 = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    ops.gemm_consume(A, B, u, rows, gates, o32, o16)
    torch.cuda.synchronize()
    scale = ref.abs().max().item()
    assert (o32 - ref).abs().max().item() / scale < 1e-4
    assert (o16.float() - ref).abs().max().item() / scale < 1e-2
    # exact arithmetic order of the routed part (products and sums rounded)
    base = torch.zeros(M, N, device=dev)
    ref0 = base.clone()
    for s in range(k):
        ref0 = ref0 + gates[:, s:s + 1] * rows[s].float()
    ref0 = u + ref0
    z32 = torch.full((M, N), float("nan"), device=dev)
    ops.consume_rows(u, rows, gates, z32)
    torch.cuda.synchronize()
    assert torch.equal(z32, ref0)


def test_gemm_rejects_internal_epilogue_kinds():
    A = torch.zeros(256, 64, device=dev, dtype=torch.bfloat16)
    B = torch.zeros(64, 64, device=dev, dtype=torch.bfloat16)
    o = torch.empty(256, 64, device=dev, dtype=torch.bfloat16)
    from paper_2411_16786_b200.errors import ContractError
    for epi in (-1, 4, 5, 6, 7, 99):
        with pytest.raises(ContractError):
            ops.gemm(epi, A, B, out_bf16=o)


@pytest.mark.parametrize("E,n,k,devices,decide", [
    (8, 8192, 2, 2, True), (8, 1000, 2, 1, False), (8, 777, 1, 4, True), (8, 300, 4, 8, False),
    (8, 37, 3, 1, True), (8, 20000, 2, 1, True), (16, 8192, 2, 8, True), (16, 1001, 2, 1, False),
    (16, 333, 5, 4, True), (16, 17, 16, 2, True), (16, 20000, 2, 1, True)])
def test_gate_route_matches_gate_then_permute(E, n, k, devices, decide):
    """dice_gate_route (gate + decide + permute in one launch, expert regions of
    cap rows) == dice_gate_topk(_decide) + dice_route_permute: ids, gates, masks,
    run counters and tile offsets identical; every expert region holds exactly
    the expert's active pairs (blocks take their offsets in arrival order, in
    pair order within a block), each row the pair's bf16 row, row_pair the
    inverse of pos, padding rows map to no pair. Repeated launches (counters
    reset by the last block) agree; 20000 rows = 625 (E = 8) / 1250 (E = 16)
    blocks, more than one resident wave."""
    hp = 256 if E == 8 else 320
    g = torch.Generator(device=dev).manual_seed(n + k)
    u = torch.randn(n, hp, device=dev, generator=g)
    wg = torch.randn(E, hp, device=dev, generator=g) * 0.1
    u16 = u.to(torch.bfloat16)
    cap = (n + 255) // 256 * 256
    state = torch.zeros(ops.route_state_words(n), dtype=torch.int64, device=dev)

    def cache_state():
        return dict(last=torch.full((n,), -10 ** 9, dtype=torch.int32, device=dev),
                    primed=torch.zeros(n, dtype=torch.uint8, device=dev),
                    red=torch.zeros(n, k, dtype=torch.uint8, device=dev),
                    cid=torch.full((n, k), -1, dtype=torch.int32, device=dev))
    st = {"route": cache_state(), "plain": cache_state()}
    for step in range(3):
        res = {}
        for mode in ("route", "plain"):
            ids = torch.empty(n, k, dtype=torch.int32, device=dev)
            gates = torch.empty(n, k, device=dev)
            act = torch.ones(n, k, dtype=torch.uint8, device=dev)
            wr = torch.zeros(n, k, dtype=torch.uint8, device=dev)
            cnt = torch.zeros(2, dtype=torch.int64, device=dev)
            pos = torch.empty(n, k, dtype=torch.int32, device=dev)
            tiles = torch.empty(E + 1, dtype=torch.int32, device=dev)
            c = st[mode]
            dec = ((step == 0, 2, ops.COND_CODES["low_score"], False, 0, c["last"], c["primed"],
                    c["red"], c["cid"], act, wr) if decide else None)
            if mode == "route":
                x_perm = torch.zeros(E * cap, hp, dtype=torch.bfloat16, device=dev)
                row_pair = torch.full((E * cap,), 777, dtype=torch.int32, device=dev)
                ops.gate_route(u, wg, k, ids, gates, x_perm, cap, pos, row_pair, tiles, cnt, state,
                               step=step, decide=dec, devices=devices, rows_total=n)
            else:
                max_rows = ops.permute_max_rows(n, k, E)
                x_perm = torch.zeros(max_rows, hp, dtype=torch.bfloat16, device=dev)
                row_pair = torch.full((max_rows,), 777, dtype=torch.int32, device=dev)
                scr = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
                ops.gate_topk(u, wg, k, ids, gates, step=step, decide=dec)
                ops.route_permute(ids, act if decide else None, u16, x_perm, pos, tiles, cnt, scr,
                                  E, devices=devices, rows_total=n, row_pair=row_pair)
            torch.cuda.synchronize()
            res[mode] = (ids, gates, act, wr, cnt, pos, tiles, x_perm, row_pair)
        a, b = res["route"], res["plain"]
        for x, y in zip(a[:5], b[:5]):
            assert torch.equal(x, y)
        assert torch.equal(a[6], b[6])
        tiles = b[6].cpu().numpy()
        pa, pb = a[5].cpu().numpy(), b[5].cpu().numpy()
        idn = b[0].cpu().numpy()
        assert np.array_equal(pa < 0, pb < 0)
        v = pb >= 0
        # the region of expert e holds rows [e*cap, e*cap + count_e): a permutation
        off = pa[v] - idn[v] * cap
        counts = np.bincount(idn[v], minlength=E)
        assert (off >= 0).all() and (off < counts[idn[v]]).all()
        for e in range(E):
            oe = np.sort(off[idn[v] == e])
            assert np.array_equal(oe, np.arange(counts[e]))
            assert tiles[e + 1] - tiles[e] == (counts[e] + 255) // 256
        assert torch.equal(a[7][torch.as_tensor(pa[v], device=dev).long()],
                           b[7][torch.as_tensor(pb[v], device=dev).long()])
        rpa = a[8].cpu().numpy()
        pair_idx = np.nonzero(v.reshape(-1))[0]
        assert np.array_equal(rpa[pa.reshape(-1)[pair_idx]], pair_idx)
        for e in range(E):   # padding up to the region's last 256-row tile
            pad = rpa[e * cap + counts[e]: e * cap + (counts[e] + 255) // 256 * 256]
            assert (pad == -1).all()
        for e in range(E):
            cnt_e = int(((idn == e) & v).sum())
            pad_end = (tiles[e + 1] - tiles[e]) * 256
            assert (rpa[e * cap + cnt_e:e * cap + pad_end] == -1).all()

