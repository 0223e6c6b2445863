"""Run one BASELINE configuration end to end on cuda:0 (CUDA-graph replay) and
report img/s, per-MoE-layer us, the staleness histogram and finiteness.
  python tools/run_config.py --preset g-16e2a [--batch 8] [--tokens 1024] [--steps 50]
  python tools/run_config.py --preset xl2-8e2a --tokens 1024 --batch 8     (C4, 512px)
"""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2411_16786_b200 as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="g-16e2a")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--tokens", type=int, default=None)
ap.add_argument("--steps", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--strategy", default="interweaved")
args = ap.parse_args()
over = {}
if args.batch:
    over["batch"] = args.batch
if args.tokens:
    over["num_tokens"] = args.tokens
if args.steps:
    over["num_steps"] = args.steps
cfg = D.preset(args.preset, **over)
t0 = time.time()
model = D.init_model(cfg, seed=0)
torch.cuda.synchronize()
t_init = time.time() - t0
x0 = D.sample_x0(cfg, 1)
runner = D.DeviceRunner(model, x0, D.Strategy(args.strategy), D.dice_policy(),
                        D.ClusterConfig(num_devices=1), 1)
runner.capture()
runner.launch()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    runner.launch()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.reps
res = runner.finish()
fin = res.final.values
print(json.dumps({
    "preset": args.preset, "config": {k: getattr(cfg, k) for k in ("num_layers", "num_experts",
                                                                    "hidden_dim", "expert_dim",
                                                                    "num_tokens", "batch",
                                                                    "num_steps")},
    "rows": cfg.total_rows, "weights_gb": sum(t.numel() * t.element_size() for lw in model.layers
                                              for t in (lw.w_mix_t, lw.w1_t, lw.w2_t, lw.ws1_t,
                                                        lw.ws2_t) if t is not None) / 1e9,
    "init_s": round(t_init, 2), "ms_per_run": ms, "img_per_s": cfg.batch / (ms / 1e3),
    "moe_layer_us": ms * 1e3 / (cfg.num_steps * cfg.num_layers),
    "finite": bool(torch.isfinite(fin).all().item()), "max_abs": float(fin.abs().max().item()),
    "staleness": res.staleness_histogram(), "active_pairs": res.active_pairs,
    "total_pairs": res.total_pairs}))
