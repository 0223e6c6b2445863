"""Worker for the 2-process expert-parallel GPU test (both ranks may share one GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def policy_by_name(D, name):
    """Policies of the EP parity cases (shared with tests/test_gpu_ep.py)."""
    import dataclasses
    dice = D.dice_policy(refresh_interval=2, warmup=2, period=3)
    return {"neutral": D.NEUTRAL, "dice": dice,
            # Random: the kept slot is drawn per GLOBAL row (policies.py:107-115)
            "random": dataclasses.replace(dice, cond_strategy=D.CondStrategy.RANDOM,
                                          sync_strategy=D.SyncStrategy.STAGGERED),
            "high_strict": dataclasses.replace(dice, cond_strategy=D.CondStrategy.HIGH_SCORE,
                                               strict_refresh=True,
                                               sync_strategy=D.SyncStrategy.SHALLOW)}[name]


def run(rank, world, port, cfg_kwargs, strategy, policy_name, out_path, same_device):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2411_16786_b200 as D
    from paper_2411_16786_b200.ep import EPRunner, sample_x0_shard
    from paper_2411_16786_b200.cluster import shard_rows

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0 if same_device else rank)
    cfg = D.ModelConfig(**cfg_kwargs)
    El = cfg.num_experts // world
    model = D.init_model(cfg, seed=5, experts=(rank * El, (rank + 1) * El))
    rows = shard_rows(cfg.total_rows, world, rank)
    x0 = sample_x0_shard(cfg, 5, rows)
    policy = policy_by_name(D, policy_name)
    r = EPRunner(model, x0, D.Strategy(strategy), policy, D.ClusterConfig(num_devices=world), 5,
                 rank=rank, world=world, time_waits=True)
    res = r.run()
    # second run through a captured graph must reproduce the first exactly
    first = res.final.values.cpu().numpy()
    r.capture()
    r.launch()
    res2 = r.finish()
    second = res2.final.values.cpu().numpy()
    out = dict(final=first, final_graph=second, rows=np.array(rows),
               staleness=np.array([(s.layer, s.used_step, s.generated_step) for s in res.staleness_records]),
               bytes=np.array([res.dispatch_bytes, res.combine_bytes]),
               pairs=np.array([res.active_pairs, res.total_pairs]),
               per_step=np.array(res.per_step_active_pairs), peak=np.array(res.peak_buffer_bytes),
               exposed=np.array(res.timeline["exposed_comm_seconds"]))
    np.savez(f"{out_path}.rank{rank}.npz", **out)
    r.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import json
    a = json.loads(sys.argv[1])
    run(**a)
