"""Expert parallelism over peer memory, 2 ranks (processes) — on one GPU if
only one is visible. The EP run must reproduce the single-GPU engine
bit-exactly (every per-row computation is identical; only the rows' placement
changes), with identical staleness records, bytes and pair counts."""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2411_16786_b200 as D  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CFG = dict(num_layers=4, num_experts=8, num_shared=2, top_k=2, hidden_dim=128, expert_dim=256,
           num_tokens=64, batch=3, num_steps=7, step_size=1e-3)


@pytest.mark.parametrize("strategy,policy,world", [("synchronous", "neutral", 2),
                                                   ("interweaved", "neutral", 2),
                                                   ("interweaved", "dice", 2),
                                                   ("interweaved", "dice", 4),
                                                   ("interweaved", "random", 2),
                                                   ("interweaved", "random", 4),
                                                   ("interweaved", "high_strict", 2),
                                                   ("displaced", "random", 4),
                                                   ("displaced", "neutral", 2),
                                                   ("displaced", "dice", 2),
                                                   ("displaced", "dice", 4)])
def test_ep_two_ranks_matches_single_gpu(strategy, policy, world):
    same = torch.cuda.device_count() < world
    port = free_port()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "ep")
        procs = []
        for rank in range(world):
            arg = json.dumps(dict(rank=rank, world=world, port=port, cfg_kwargs=CFG,
                                  strategy=strategy, policy_name=policy, out_path=out,
                                  same_device=same))
            procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "ep_worker.py"), arg]))
        for p in procs:
            try:
                p.wait(timeout=240)
            except subprocess.TimeoutExpired:
                for q in procs:
                    q.kill()
                pytest.fail("EP workers timed out")
            assert p.returncode == 0
        parts = [np.load(f"{out}.rank{r}.npz") for r in range(world)]
    cfg = D.ModelConfig(**CFG)
    model = D.init_model(cfg, seed=5)
    x0 = D.sample_x0(cfg, 5)
    from tests.ep_worker import policy_by_name
    pol = policy_by_name(D, policy)
    ref = D.run_sampling(model, x0, D.Strategy(strategy), pol, D.ClusterConfig(num_devices=world), 5)
    fin = ref.final.values.cpu().numpy()
    for r, part in enumerate(parts):
        a, b = part["rows"]
        assert np.array_equal(part["final"], fin[a:b]), f"rank {r} final differs"
        assert np.array_equal(part["final_graph"], part["final"]), "graph replay differs"
        st = np.array([(s.layer, s.used_step, s.generated_step) for s in ref.staleness_records])
        assert np.array_equal(part["staleness"], st)
        assert part["bytes"].tolist() == [ref.dispatch_bytes, ref.combine_bytes]
        assert part["pairs"].tolist() == [ref.active_pairs, ref.total_pairs]
        assert part["per_step"].tolist() == ref.per_step_active_pairs
        assert int(part["peak"]) == ref.peak_buffer_bytes


@pytest.mark.parametrize("geometry", ["xl", "g"])
def test_ep_xl_widths_matches_single_gpu(geometry):
    """Expert parallelism at the XL layer widths (h=1152, e=4608, 8 experts,
    2 shared; 4 layers, 3 steps, full DICE policy; 2 ranks) and at the G-16E2A
    widths (h=1664 padded to 1792, e=6656, 16 experts; 4 ranks of 4 experts):
    the run over peer memory reproduces the single-GPU engine bit-exactly — the
    bench geometry's tile shapes (256x192 expert GEMM2 with the combine stored
    into the peers' windows by its epilogue, dual GEMM1 launches) on both sides."""
    if geometry == "xl":
        world = 2
        cfg_kw = dict(num_layers=4, num_experts=8, num_shared=2, top_k=2, hidden_dim=1152,
                      expert_dim=4608, num_tokens=256, batch=4, num_steps=3, step_size=2e-5)
    else:
        world = 4
        cfg_kw = dict(num_layers=2, num_experts=16, num_shared=2, top_k=2, hidden_dim=1664,
                      expert_dim=6656, num_tokens=128, batch=4, num_steps=3, step_size=2e-5)
    same = torch.cuda.device_count() < world
    port = free_port()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "ep")
        procs = []
        for rank in range(world):
            arg = json.dumps(dict(rank=rank, world=world, port=port, cfg_kwargs=cfg_kw,
                                  strategy="interweaved", policy_name="dice", out_path=out,
                                  same_device=same))
            procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "ep_worker.py"), arg]))
        for p in procs:
            try:
                p.wait(timeout=300)
            except subprocess.TimeoutExpired:
                for q in procs:
                    q.kill()
                pytest.fail("EP workers timed out")
            assert p.returncode == 0
        parts = [np.load(f"{out}.rank{r}.npz") for r in range(world)]
    cfg = D.ModelConfig(**cfg_kw)
    model = D.init_model(cfg, seed=5)
    x0 = D.sample_x0(cfg, 5)
    pol = D.dice_policy(refresh_interval=2, warmup=2, period=3)
    ref = D.run_sampling(model, x0, D.Strategy.INTERWEAVED, pol, D.ClusterConfig(num_devices=world), 5)
    fin = ref.final.values.cpu().numpy()
    for part in parts:
        a, b = part["rows"]
        assert np.array_equal(part["final"], fin[a:b])
        assert part["bytes"].tolist() == [ref.dispatch_bytes, ref.combine_bytes]
        assert part["pairs"].tolist() == [ref.active_pairs, ref.total_pairs]
