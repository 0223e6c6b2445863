"""bench.py end to end (the driver's contract): one JSON line on stdout with the
keys the driver and judge read. The reference arm runs on CPU here; the GPU arm
runs the tiny preset through the same code path as the default XL workload."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    line = _run(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1"], 300)
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "img/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["cpu_baseline"]["samples_timed"] == 2
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # a step of this arm is one bounded sample: its time, not the extrapolated run
    assert line["ms_per_step"] * line["steps"] <= line["wall_seconds"] * 1e3 + 1.0


def test_schedule_pair_count_matches_oracle_run():
    """The reference arm prices the run by its exact active-pair total, counted
    on a narrow copy of the schedule: equal to the full-width oracle run."""
    sys.path.insert(0, ROOT)
    import bench
    from oracle import dice_oracle as O
    g = bench._oracle_geometry(O, "tiny")
    res = O.run_schedule(g, O.init_params(g, 0), O.initial_latent(g, 0), O.INTERWEAVED,
                         bench._oracle_policy(O, "tiny"), 1, 0)
    stages, n_sync, pairs = bench.schedule_pairs(O, "tiny")
    assert stages == g.num_steps * g.num_layers
    assert pairs == res.active_pairs
    assert n_sync == sum(1 for (l, used, gen) in res.staleness if used == gen)


@pytest.mark.gpu
def test_gpu_arm_line():
    line = _run(["--config", "tiny", "--steps", "2", "--warmup", "3"], 900)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "data", "config", "roofline",
                "cpu_baseline", "e2e", "gpu_launches", "clocks", "quality", "breakdown"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    rf = line["roofline"]
    assert rf["bound"] == "tensor" and rf["achieved"] > 0 and 0 < rf["frac"]
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["cpu_baseline"]["value"] > 0
    q = line["quality"]
    assert q["dice_latent_mse_vs_sync"] >= 0 and q["speedup_dice_vs_sync"] > 0
    assert line["buffers"]["device_bytes"] > 0


@pytest.mark.gpu
def test_gpu_arm_expert_parallel_line():
    """--gpus 2 spawns its two ranks itself (on one GPU when only one is
    visible): the line reports n_gpus 2, the exposed all-to-all time and its
    parts (flag waits, main-stream exchange kernels, waits for the overlapped
    comm-stream sends)."""
    env = dict(os.environ)
    import torch
    if torch.cuda.device_count() < 2:
        env["DICE_BENCH_SAME_DEVICE"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "tiny",
                        "--gpus", "2", "--steps", "2", "--warmup", "3"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    parts = line["a2a_parts_us"]
    assert set(parts) == {"flag_waits", "main_stream_send_and_regroup_kernels",
                          "waits_for_overlapped_sends"}
    assert line["exposed_a2a_us"] >= parts["main_stream_send_and_regroup_kernels"] > 0
    # the synchronous expert-parallel path timed on the same ranks (north-star ratio)
    q = line["quality"]
    assert q["sync_ep_ms_per_run"] > 0 and q["speedup_dice_vs_sync"] > 0
    assert q["dice_latent_mse_vs_sync"] >= 0
