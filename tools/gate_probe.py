"""Isolated timings of the router launches on the bench geometry (XL, 8192
rows, hp = 1152, E = 8, k = 2; CUDA events, median of reps):
gate (+ decision) alone, gate + decision + permute (dice_gate_route), the
three-kernel permute, and each right behind the local GEMM that produces u
(as in the step). python tools/gate_probe.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_16786_b200 as D  # noqa: E402
from paper_2411_16786_b200 import ops  # noqa: E402

cfg = D.preset("xl2-8e2a", batch=32, num_steps=2, num_layers=2)
model = D.init_model(cfg, seed=0)
x0 = D.sample_x0(cfg, 1000)
r = D.DeviceRunner(model, x0, D.Strategy.INTERWEAVED, D.dice_policy(),
                   D.ClusterConfig(num_devices=1), 1000)
r.launch()
torch.cuda.synchronize()
lw = model.layers[1]
p = r.payloads[0]
n, k = r.n, r.k


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def dec():
    return r.cache.decide_args(1, 7, r.policy, False, p.active, p.write)


def gate():
    ops.gate_topk(r.u32, lw.w_gate_t, k, p.ids, p.gates, None, r.status, 7, 1, decide=dec())


def route():
    ops.gate_route(r.u32, lw.w_gate_t, k, p.ids, p.gates, p.x_perm, r.cap, p.pos, p.row_pair,
                   p.tiles, r.counters[1, 1], r.route_state, None, r.status, 7, 1, decide=dec(),
                   devices=1, rows_total=n)


def permute3():
    ops.route_permute(p.ids, p.active, r.u16, p.x_perm, p.pos, p.tiles, r.counters[1, 1],
                      r.scratch, r.E, devices=1, row0=0, rows_total=n, row_pair=p.row_pair)


def local():
    ops.gemm(ops.EPI_GELU_RESID, r.h16, lw.w_mix_t, out_f32=r.u32, out_bf16=r.u16, residual=r.h32)


res = {}
res["local"] = timed(local)
res["gate+decide"] = timed(gate)
res["gate_route"] = timed(route)
res["permute(3 kernels)"] = timed(permute3)
res["local->gate+decide"] = timed(lambda: (local(), gate())) - res["local"]
res["local->gate_route"] = timed(lambda: (local(), route())) - res["local"]
bytes_gate = 4 * n * 1152
print({k_: round(v, 2) for k_, v in res.items()})
print(f"gate+decide alone: {bytes_gate / res['gate+decide'] / 1e3:.0f} GB/s of u reads")
