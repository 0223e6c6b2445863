import os, sys
sys.path.insert(0, ".")
import torch
import paper_2411_16786_b200 as D
CFG = dict(num_layers=4, num_experts=8, num_shared=2, top_k=2, hidden_dim=128, expert_dim=256,
           num_tokens=64, batch=3, num_steps=7, step_size=1e-3)
cfg = D.ModelConfig(**CFG)
model = D.init_model(cfg, seed=5)
x0 = D.sample_x0(cfg, 5)
pol = D.dice_policy(refresh_interval=2, warmup=2, period=3)
for f in ("1", "0"):
    os.environ["DICE_FUSED_GATE"] = f
    r = D.DeviceRunner(model, x0, D.Strategy.INTERWEAVED, pol, D.ClusterConfig(num_devices=2), 5)
    res = r.run()
    print(f, res.dispatch_bytes, res.combine_bytes, res.active_pairs, res.per_step_active_pairs, float(res.final.values.abs().sum()))
    print(r.counters[:, :, 1].cpu().numpy().tolist())
