"""Per-op device time inside the bench step (XL, 32 images, full DICE, CUDA-graph
replay, power-capped clocks as in bench.py). Every library op the runner calls
is bracketed by graph-safe CUDA events; prints total us per op kind per run
and per MoE layer-stage.  python tools/kernel_breakdown.py [--overlap]"""
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
import paper_2411_16786_b200 as D  # noqa: E402
from paper_2411_16786_b200 import ops, schedules  # noqa: E402

EPI = {0: "store_bf16", 1: "gelu_bf16", 2: "store_f32", 3: "gelu_resid"}
records = []
pool = []


def wrap(name, fn, labeler=None):
    def inner(*a, **k):
        i = len(records)
        if i >= len(pool):
            pool.append((ops.DeviceEvent(), ops.DeviceEvent()))
        e0, e1 = pool[i]
        e0.record()
        r = fn(*a, **k)
        e1.record()
        records.append((labeler(*a, **k) if labeler else name, e0, e1))
        return r
    return inner


def gemm_label(epi, A, B, **kw):
    return f"gemm {EPI[epi]} {A.shape[0]}x{B.shape[0]}x{A.shape[1]}"


for name in ("gate_topk", "route_permute", "denoise", "expert_gemm1_with_shared",
             "expert_gemm2_pairs", "gemm_consume"):
    setattr(ops, name, wrap(name, getattr(ops, name)))
ops.gemm = wrap("gemm", ops.gemm, gemm_label)
_decide = D.policies.TokenCache.decide_into
D.policies.TokenCache.decide_into = wrap("cond_decide", _decide)

cfg = D.preset("xl2-8e2a", batch=32)
model = D.init_model(cfg, seed=0)
x0 = D.sample_x0(cfg, 1000)
r = D.DeviceRunner(model, x0, D.Strategy.INTERWEAVED, D.dice_policy(), D.ClusterConfig(num_devices=1),
                   1000, overlap="--overlap" in sys.argv)
r.capture()
n_cap = len(records)
for _ in range(3):
    r.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r.launch()
e1.record()
torch.cuda.synchronize()
total = e0.elapsed_time(e1)
# the captured records are the second launch() inside capture() (warm-up first)
recs = records[n_cap // 2:n_cap]
agg = defaultdict(lambda: [0.0, 0])
for lab, a, b in recs:
    t = a.elapsed_ms(b)
    agg[lab][0] += t
    agg[lab][1] += 1
stages = cfg.num_steps * cfg.num_layers
print(f"run {total:.1f} ms, {32 / total * 1e3:.2f} img/s, {total * 1e3 / stages:.1f} us per layer-stage")
s = 0.0
for lab, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    s += t
    print(f"{lab:40s} {t:8.2f} ms  x{c:5d}  avg {t / c * 1e3:8.1f} us  per-stage {t * 1e3 / stages:7.1f} us")
print(f"sum of bracketed ops {s:.1f} ms ({s / total:.3f} of the run)")
