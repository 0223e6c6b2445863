"""The G-16E2A router (E = 16, hp = 1792, 8192 rows) in isolation, for an ncu
capture of gate4_topk_kernel<16, ...>: three launches, the last one profiled
(`ncu --set full -k regex:gate4 -s 2 -c 1 python tools/profile_router_g.py`);
also prints its CUDA-event time."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_16786_b200 as D  # noqa: E402
from paper_2411_16786_b200 import ops  # noqa: E402

cfg = D.preset("g-16e2a", num_tokens=1024, batch=8, num_steps=2, num_layers=1)
model = D.init_model(cfg, seed=0)
x0 = D.sample_x0(cfg, 1000)
r = D.DeviceRunner(model, x0, D.Strategy.INTERWEAVED, D.dice_policy(),
                   D.ClusterConfig(num_devices=1), 1000)
r.launch()
torch.cuda.synchronize()
lw = model.layers[0]
p = r.payloads[0]
u = torch.randn_like(r.u32)


def route():
    ops.gate_route(u, lw.w_gate_t, r.k, p.ids, p.gates, p.x_perm, r.cap, p.pos, p.row_pair,
                   p.tiles, r.counters[1, 0], r.route_state, None, r.status, 1, 0,
                   decide=r.cache.decide_args(0, 1, r.policy, False, p.active, p.write),
                   devices=1, rows_total=r.n)


for _ in range(3):
    route()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); route(); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(f"G router (E = 16, hp = {r.hp}, {r.n} rows): {ts[len(ts) // 2]:.1f} us")
