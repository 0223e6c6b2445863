"""Small eager workload touching every kernel of the library, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
tools/sanitize.sh runs it under each tool. E = 8 runs go through the fused
gate + decide + permute launch (dice_gate_route); E = 16 through the gate +
three-kernel permute; the functional API covers cache assemble, combine,
consume rows and the step-similarity reductions. No CUDA graph (the sanitizer
reports per launch)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2411_16786_b200 as D  # noqa: E402

torch.cuda.set_device(0)


def run(E, strategy, policy, devices=2, steps=5):
    cfg = D.ModelConfig(num_layers=3, num_experts=E, num_shared=2, top_k=2, hidden_dim=128,
                        expert_dim=256, num_tokens=64, batch=2, num_steps=steps, step_size=1e-3)
    model = D.init_model(cfg, seed=3)
    res = D.run_sampling(model, D.sample_x0(cfg, 3), strategy, policy,
                         D.ClusterConfig(num_devices=devices), 3, track_similarity=True)
    torch.cuda.synchronize()
    return res


pol = D.dice_policy(refresh_interval=2, warmup=1, period=3)
rnd = D.PolicyConfig(sync_strategy=D.SyncStrategy.STAGGERED, cond_strategy=D.CondStrategy.RANDOM,
                     refresh_interval=2, warmup=1, period=3, strict_refresh=True)
for E in (8, 16):
    for st in (D.Strategy.SYNCHRONOUS, D.Strategy.INTERWEAVED, D.Strategy.DISPLACED):
        run(E, st, pol)
    run(E, D.Strategy.INTERWEAVED, rnd)

# functional API: routed_rows / combine_outputs / TokenCache.assemble paths
cfg = D.ModelConfig(num_layers=1, num_experts=8, num_shared=2, top_k=2, hidden_dim=96,
                    expert_dim=192, num_tokens=40, batch=1, num_steps=2, step_size=1e-3)
model = D.init_model(cfg, seed=1)
x = D.sample_x0(cfg, 1)
u = D.local_block(model, 0, x)
r = D.gate(model, 0, u)
rows = D.routed_rows(model, 0, u.values, r)
sh = D.shared_forward(model, 0, u)
out = D.combine_outputs(r, rows, sh, r)
cache = D.TokenCache(1, cfg.total_rows, 2, cfg.hidden_dim, device="cuda")
act, wr = cache.decide(0, 0, r, pol, force_refresh=True)
cache.assemble(0, rows, r, act, wr)
act, wr = cache.decide(0, 1, r, pol)
cache.assemble(0, rows, r, act, wr)
torch.cuda.synchronize()
print("sanitize_ops done")
