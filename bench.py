"""Benchmark of the B200-native DICE sampling path (BASELINE.json metric).

Default workload (BASELINE configs[2], restated at the SURVEY.md §8 XL preset):
DiT-MoE-XL/2-8E2A toy geometry (L=28, E=8, S=2, k=2, h=1152, e=4608),
256 px = 256 tokens/image, 32 images per GPU, 50 denoising steps of
x <- x - eta*h, full DICE = interweaved + Deep selective sync + LowScore
conditional communication (R=5) + warmup 6 / period 10. Synthetic latents
and random-init weights from the reference's splitmix64 streams.
``--config`` selects the other BASELINE configurations (s256 = configs[1],
xl512 = configs[3], g512 = configs[4]) and ``tiny`` (the test preset).

One bench "step" = one full 50-step sampling run of the per-GPU batch.
value = images/s (whole job), device-timed with CUDA events (max over ranks);
e2e = the same metric through the serving call (x0 H2D from pinned host
memory, run, final latent D2H) timed around the call.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config NAME]

``--gpus N`` (N > 1) outside torchrun spawns the N ranks itself (one process
per GPU, RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1); under
torchrun it reads them from the environment.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name -> BASELINE configuration restated on the SURVEY.md §8 presets.
# images_per_gpu is fixed as N grows (weak scaling).
CONFIGS = {
    "xl256": dict(
        baseline="configs[2]", preset="xl2-8e2a", tokens=256, images_per_gpu=32, policy="dice",
        metric="DiT-MoE-XL/2 img/s (full-DICE 50-step sampling, 256px, 32 img/GPU)",
        workload=("DiT-MoE-XL/2-8E2A toy geometry (L=28,E=8,S=2,k=2,h=1152,e=4608), 256 tok/img, "
                  "32 img/GPU, 50-step full-DICE sampling (interweaved+Deep sync+LowScore R=5, "
                  "W=6, P=10)")),
    "s256": dict(
        baseline="configs[1]", preset="s2-8e2a", tokens=256, images_per_gpu=16, policy="neutral",
        steps=50,
        metric="DiT-MoE-S/2 img/s (interweaved 50-step sampling, 256px, 16 img/GPU)",
        workload=("DiT-MoE-S/2-8E2A toy geometry (L=12,E=8,S=2,k=2,h=384,e=1536), 256 tok/img, "
                  "16 img/GPU, 50-step interweaved sampling (no selective sync / cond comm)")),
    "xl512": dict(
        baseline="configs[3]", preset="xl2-8e2a", tokens=1024, images_per_gpu=8, policy="dice",
        metric="DiT-MoE-XL/2 img/s (full-DICE 50-step sampling, 512px, 8 img/GPU)",
        workload=("DiT-MoE-XL/2-8E2A toy geometry (L=28,E=8,S=2,k=2,h=1152,e=4608), 1024 tok/img "
                  "(512px), 8 img/GPU, 50-step full-DICE sampling with conditional communication")),
    "g512": dict(
        baseline="configs[4]", preset="g-16e2a", tokens=1024, images_per_gpu=8, policy="dice",
        metric="DiT-MoE-G img/s (full-DICE 50-step sampling, 512px, 8 img/GPU)",
        workload=("DiT-MoE-G-16E2A toy geometry (L=40,E=16,S=2,k=2,h=1664 padded to 1792,e=6656), "
                  "1024 tok/img (512px), 8 img/GPU, 50-step full-DICE sampling")),
    "tiny": dict(
        baseline="test preset", preset=None, tokens=64, images_per_gpu=2, policy="dice_small",
        metric="tiny DICE img/s (test preset)",
        workload="test preset (L=4,E=8,S=2,k=2,h=128,e=256), 64 tok/img, 2 img/GPU, 6 steps",
        geometry=dict(num_layers=4, num_experts=8, num_shared=2, top_k=2, hidden_dim=128,
                      expert_dim=256, num_steps=6, step_size=1e-3)),
}


def model_config(D, name, world=1):
    c = CONFIGS[name]
    batch = c["images_per_gpu"] * world
    if c["preset"] is None:
        return D.ModelConfig(**c["geometry"], num_tokens=c["tokens"], batch=batch)
    over = dict(num_tokens=c["tokens"], batch=batch)
    if "steps" in c:
        over["num_steps"] = c["steps"]
    return D.preset(c["preset"], **over)


def policy_of(D, name):
    p = CONFIGS[name]["policy"]
    if p == "dice":
        return D.dice_policy()
    if p == "dice_small":
        return D.dice_policy(refresh_interval=2, warmup=2, period=3)
    return D.NEUTRAL


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops_sustained"], p["hbm_gbs"], "measured"
    except Exception:
        return 1400.0, 6650.0, "fallback"


def csrc_digest() -> str:
    """sha256 over the CUDA sources: ties a committed ncu traffic capture to the
    kernels it was taken on."""
    d = os.path.join(ROOT, "paper_2411_16786_b200", "csrc")
    h = hashlib.sha256()
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def measured_traffic(config):
    """DRAM bytes (ncu --set full) of the roofline kernel, from the committed
    capture, only when it was taken on the current kernel sources."""
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except Exception:
        return None, "no committed capture"
    if t.get("config") != config:
        return None, f"capture is for config {t.get('config')!r}"
    if t.get("csrc_sha") != csrc_digest():
        return None, "stale: the committed capture predates the current kernel sources"
    return t["traffic_bytes_per_launch_pair"], t.get("capture", "")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,power.limit")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})

        def num(i):
            out = []
            for r in self.rows:
                try:
                    out.append(float(r[i]))
                except (IndexError, ValueError):
                    pass
            return out
        pw, pl = num(7), num(8)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w": statistics.median(pw) if pw else None,
                "power_limit_w": max(pl) if pl else None,
                "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- CPU oracle
_CPU_STATE = {}


def _oracle_geometry(O, name):
    c = CONFIGS[name]
    if c["preset"] is None:
        geo = dict(c["geometry"])
    else:
        geo = dict(O.PRESETS[c["preset"]])
        geo.setdefault("num_steps", c.get("steps", 50))
    geo["num_tokens"] = c["tokens"]
    return O.Geometry(**{**geo, "batch": c["images_per_gpu"]})


def _oracle_policy(O, name):
    p = CONFIGS[name]["policy"]
    if p == "dice":
        return O.dice_defaults()
    if p == "dice_small":
        return O.dice_defaults(refresh_interval=2, warmup=2, period=3)
    return O.Policy()


def schedule_pairs(O, name):
    """(stages, sync stages, active pairs) of the interweaved run of ``name`` at
    its full row count. The active-pair cadence of the configurations' policies
    (LowScore non-strict, or none) does not depend on the routed values and is
    identical for every token, so the oracle schedule run on a few rows of a
    tiny width counts it exactly; the count scales with the rows."""
    g = _oracle_geometry(O, name)
    small = O.Geometry(**{**g.__dict__, "hidden_dim": 4, "expert_dim": 4, "num_tokens": 8,
                          "batch": 1})
    pol = _oracle_policy(O, name)
    res = O.run_schedule(small, O.init_params(small, 0), O.initial_latent(small, 0),
                         O.INTERWEAVED, pol, 1, 0)
    sync_set = O.sync_layer_set(pol.sync_strategy, g.num_layers, pol.explicit_layers)
    n_sync = sum(1 for s in range(g.num_steps) for l in range(g.num_layers)
                 if s == 0 or O.sync_step(s, pol.warmup, pol.period) or l in sync_set)
    scale = g.total_rows // small.total_rows
    return g.num_steps * g.num_layers, n_sync, res.active_pairs * scale


def cpu_sample(name, threads_note: str):
    """The reference algorithm (oracle: numpy fp64 restatement of dicesim) timed
    on a bounded sample of the same workload: one synchronous MoE-layer stage
    (all k pairs per token) and one interweaved conditional-communication stage
    (only the pairs the LowScore cadence keeps active, stale-cache assemble) at
    the configuration's full geometry and rows. Stage cost is affine in the
    active pairs, t = a + b*P, so the two samples price every stage of the run;
    the run's exact active-pair total comes from schedule_pairs(). Weight
    generation is excluded (weights are resident on the GPU side too)."""
    import numpy as np
    from oracle import dice_oracle as O
    g = _oracle_geometry(O, name)
    pol = _oracle_policy(O, name)
    if name not in _CPU_STATE:
        x = O.initial_latent(g, 0)
        p = O.init_layer(g, 0, 0)
        _CPU_STATE[name] = (x, p, schedule_pairs(O, name))
    x, p, (n_stages, n_sync, pairs_total) = _CPU_STATE[name]
    n, k = g.total_rows, g.top_k
    cache = O.CadenceCache(1, n, k, g.hidden_dim)

    def stage(step, force):
        t0 = time.perf_counter()
        u = O.mixing_block(p, x)
        r = O.route_tokens(u, p.w_gate, k)
        active, write = cache.decide(0, step, r.ids, pol, force)
        rows = O.expert_rows(p, u, r, active)
        gates = r.gates
        if pol.cond_strategy != O.COND_OFF:
            rows, gates = cache.assemble(0, rows, r, active, write)
        out = u + O.weighted_combine(rows, O.shared_sum(p, u), gates)
        dt = time.perf_counter() - t0
        assert np.isfinite(out).all()
        return dt, int(np.count_nonzero(active))

    t_sync, p_sync = stage(0, True)
    t_async, p_async = stage(1, False)
    if p_async < p_sync:
        b = max(t_sync - t_async, 0.0) / (p_sync - p_async)
    else:                      # no conditional communication: every stage moves all pairs
        b = t_sync / p_sync
    a = t_sync - b * p_sync
    run_seconds = n_stages * a + b * pairs_total
    imgs = g.batch
    return {
        "value": imgs / run_seconds, "unit": "img/s", "cores": os.cpu_count(), "kind": "port",
        "sample": (f"1 synchronous + 1 conditional-communication MoE-layer stage (local+gate+"
                   f"decide+routed experts on active pairs+assemble+shared+combine) at full "
                   f"geometry, {n} rows, fp64 numpy/OpenBLAS ({threads_note}): "
                   f"{t_sync:.2f} s / {p_sync} pairs and {t_async:.2f} s / {p_async} pairs; "
                   f"run = {n_stages} stages, {pairs_total} active pairs "
                   f"({n_sync} synchronous stages) priced at a + b*pairs"),
        "sample_seconds": t_sync + t_async,
        "run_seconds_extrapolated": run_seconds,
    }


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    cores = os.cpu_count()
    vals = []
    # each step = one bounded sample (one sync + one DICE stage at full geometry);
    # at most one warm-up sample
    t_start = time.perf_counter()
    for i in range(min(args.warmup, 1) + args.steps):
        s = cpu_sample(args.config, f"{cores} host threads")
        if i >= min(args.warmup, 1):
            vals.append(s)
    wall = time.perf_counter() - t_start
    v = statistics.median([s["value"] for s in vals])
    ms_sample = statistics.mean([s["sample_seconds"] for s in vals]) * 1e3
    line = {
        "impl": "reference", "metric": cfg["metric"], "value": v, "unit": "img/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # one bench step of this arm is one bounded CPU sample (its measured time)
        "ms_per_step": ms_sample, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "parallelism": "cpu", "baseline": cfg["baseline"]},
        "cpu_baseline": {"value": v, "unit": "img/s", "cores": cores, "kind": "port",
                         "sample": vals[0]["sample"], "samples_timed": len(vals)},
        "e2e": {"value": v, "unit": "img/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_seconds": wall,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm
def op_breakdown(D, model, x0, policy, cluster, seed, cfg, args):
    """Per-op device time of one graph replay of the bench run, with graph-safe
    CUDA events around every library op, and each op's achieved rate against
    its roofline: HBM-bound ops in GB/s of algorithmic bytes over the measured
    HBM copy bandwidth, GEMMs in TFLOP/s over the sustained bf16 peak.
    Algorithmic bytes / FLOPs per call (R rows, h hidden, e expert width, k slots,
    E experts, S shared, P active pairs of that (step, layer) from the device
    counters):
      gate_decide     4Rh (u) + 4Eh (W_gate) + 8Rk (ids, gates) + 5R + 3Rk (cache state)
      gate_route      gate_decide + 2hP (bf16 rows to their permuted positions) + 8P (pos,
                      row_pair)
      permute         4hP (row gather read + write, bf16) + 9Rk (ids, masks, positions)
      cache_assemble  2hP (fresh rows) + 2h(Rk - P) (cached rows) + 4Rh (combine slot) + 10Rk
                      (cache-row writes of refreshed pairs not counted: a lower bound)
      denoise         14Rh
      local_gemm      2Rh^2;  shared_gemm1 / shared_gemm2_consume 2RhSe each;  grouped_ffn 4heP
      (grouped_ffn+shared_gemm1: the expert FFN launches that also carry the stage's
       shared GEMM1, 4heP + 2RhSe)
    A GEMM also moves algorithmic bytes (operands once, epilogue inputs / outputs):
      local_gemm      2Rh (A) + 2h^2 (W_mix) + 4Rh (residual) + 6Rh (u f32 + bf16)
      shared_gemm1    2Rh + 2hSe + 2RSe
      shared_gemm2_consume  2RSe + 2hSe + 4Rh (u) + 2kRh (token-cache rows) + 4Rk + 6Rh
      grouped_ffn     2hP + 2Ehe + 2eP (GEMM1) + 2eP + 2Ehe + 2hP + 8P (GEMM2)
    and is bound by whichever roofline takes longer: `bound` names it, `frac` is the
    binding roofline's time over the measured time (tensor_frac / hbm_frac: each one).
    """
    import torch
    r = D.DeviceRunner(model, x0, D.Strategy.INTERWEAVED, policy, cluster, seed, time_ops=True,
                       overlap=args.overlap)
    if not args.eager:
        r.capture()
    r.launch()
    r.launch()
    torch.cuda.synchronize()
    times = r.op_times()
    cnt = r.counters.cpu().numpy()
    del r
    torch.cuda.empty_cache()
    R, h, e, k, E, S = (cfg.total_rows, cfg.hidden_dim, cfg.expert_dim, cfg.top_k,
                        cfg.num_experts, cfg.num_shared)
    peak_tf, hbm, _ = peaks()
    agg = {}
    for name, ms, step, layer in times:
        P = float(cnt[step, layer, 0]) if layer >= 0 else 0.0
        if name == "gate_decide":
            work, kind = 4 * R * h + 4 * E * h + 8 * R * k + 5 * R + 3 * R * k, "hbm"
        elif name == "gate_route":
            work, kind = (4 * R * h + 4 * E * h + 8 * R * k + 5 * R + 3 * R * k
                          + 2 * h * P + 8 * P), "hbm"
        elif name == "permute":
            work, kind = 4 * h * P + 9 * R * k, "hbm"
        elif name == "cache_assemble":
            work, kind = 2 * h * P + 2 * h * (R * k - P) + 4 * R * h + 10 * R * k, "hbm"
        elif name == "denoise":
            work, kind = 14 * R * h, "hbm"
        elif name == "local_gemm":
            work, kind = 2.0 * R * h * h, "tensor"
            byts = 12.0 * R * h + 2.0 * h * h
        elif name == "shared_gemm1":
            work, kind = 2.0 * R * h * S * e, "tensor"
            byts = 2.0 * R * h + 2.0 * h * S * e + 2.0 * R * S * e
        elif name == "shared_gemm2_consume":
            work, kind = 2.0 * R * h * S * e, "tensor"
            byts = 2.0 * R * S * e + 2.0 * h * S * e + 10.0 * R * h + 2.0 * k * R * h + 4.0 * R * k
        elif name.startswith("grouped_ffn"):
            work, kind = 4.0 * h * e * P + (2.0 * R * h * S * e if "shared" in name else 0.0), "tensor"
            byts = 4.0 * h * P + 4.0 * E * h * e + 4.0 * e * P + 8.0 * P
            if "shared" in name:
                byts += 2.0 * R * h + 2.0 * h * S * e + 2.0 * R * S * e
        else:
            continue
        if kind == "hbm":
            byts = work
        a = agg.setdefault(name, [0.0, 0, 0.0, kind, 0.0])
        a[0] += ms
        a[1] += 1
        a[2] += work
        a[4] += byts
    total_ms = sum(v[0] for v in agg.values())
    out = {}
    for name, (ms, calls, work, kind, byts) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        sec = ms * 1e-3
        hbm_frac = byts / (hbm * 1e9) / sec
        if kind == "hbm":
            out[name] = {"us_per_call": ms * 1e3 / calls, "calls": calls, "share": ms / total_ms,
                         "bound": "hbm", "achieved": byts / sec / 1e9, "unit": "GB/s",
                         "peak": hbm, "frac": hbm_frac}
            continue
        tensor_frac = work / (peak_tf * 1e12) / sec
        bound = "hbm" if hbm_frac > tensor_frac else "tensor"
        out[name] = {"us_per_call": ms * 1e3 / calls, "calls": calls, "share": ms / total_ms,
                     "bound": bound, "achieved": work / sec / 1e12, "unit": "TFLOP/s",
                     "peak": peak_tf, "achieved_gbs": byts / sec / 1e9, "hbm_peak": hbm,
                     "tensor_frac": tensor_frac, "hbm_frac": hbm_frac,
                     "frac": max(tensor_frac, hbm_frac)}
    return out


def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2411_16786_b200 as D

    conf = CONFIGS[args.config]
    rank, world, local = dist_env()
    # DICE_BENCH_SAME_DEVICE=1: every rank on cuda:0 (functional test of the EP
    # path on a one-GPU box; gloo for the host-side collectives)
    same_device = os.environ.get("DICE_BENCH_SAME_DEVICE") == "1"
    if not torch.cuda.is_available():
        raise RuntimeError("bench.py (impl b200) needs a CUDA device")
    if world > 1 and not same_device and torch.cuda.device_count() < world:
        raise RuntimeError(f"--gpus {world} needs {world} visible GPUs, "
                           f"found {torch.cuda.device_count()}")
    torch.cuda.set_device(0 if same_device else local)
    if world > 1:
        if same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if same_device else "cuda"

    def allreduce(x, op):
        t = torch.tensor(x, device=coll_dev)
        dist.all_reduce(t, op=op)
        return t.cpu()
    policy = policy_of(D, args.config)
    seed = 1000
    ipg = conf["images_per_gpu"]
    if world == 1:
        cfg = model_config(D, args.config)
        model = D.init_model(cfg, seed=0)
        x0 = D.sample_x0(cfg, seed)
        cluster = D.ClusterConfig(num_devices=1)
        runner = D.DeviceRunner(model, x0, D.Strategy.INTERWEAVED, policy, cluster, seed,
                                time_experts=True, overlap=args.overlap)
    else:
        # expert parallelism: images_per_gpu per GPU (weak scaling), experts e // (E/N)
        # per rank, token rows (t*N)//R per rank, exchange over peer memory
        from paper_2411_16786_b200.ep import EPRunner, sample_x0_shard
        from paper_2411_16786_b200.cluster import shard_rows
        cfg = model_config(D, args.config, world)
        El = cfg.num_experts // world
        model = D.init_model(cfg, seed=0, experts=(rank * El, (rank + 1) * El))
        x0 = sample_x0_shard(cfg, seed, shard_rows(cfg.total_rows, world, rank))
        cluster = D.ClusterConfig(num_devices=world)
        runner = EPRunner(model, x0, D.Strategy.INTERWEAVED, policy, cluster, seed, rank=rank,
                          world=world, time_waits=True, time_experts=True)
    if not args.eager:
        runner.capture()       # the whole 50-step run as one CUDA graph

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        runner.launch()
    runner.finish()          # raises NumericalDivergenceError on non-finite
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        e0.record()
        for _ in range(args.steps):
            runner.launch()
        e1.record()
        barrier()
    launches = runner.launches_per_run * args.steps
    ms = e0.elapsed_time(e1)
    expert_events = list(runner._expert_events)
    res = runner.finish()
    cnt = runner.counters.cpu().numpy()
    exposed_ms = wait_ms = kern_ms = join_ms = 0.0
    if world > 1:
        tl = res.timeline or {}
        # max over ranks of (flag waits + exchange kernels) on the rank's stream
        ex = allreduce([tl.get("exposed_comm_seconds", 0.0) * 1e3,
                        tl.get("comm_wait_seconds", 0.0) * 1e3,
                        tl.get("comm_kernel_seconds", 0.0) * 1e3,
                        tl.get("comm_join_seconds", 0.0) * 1e3], dist.ReduceOp.MAX)
        exposed_ms, wait_ms, kern_ms, join_ms = (float(v) for v in ex)
        cnt = allreduce(cnt, dist.ReduceOp.SUM).numpy()
    if world > 1:
        ms = float(allreduce([ms], dist.ReduceOp.MAX).item())
    ms_per_step = ms / args.steps
    value = world * ipg * args.steps / (ms / 1e3)

    # roofline: grouped expert FFN (GEMM1 gelu + GEMM2), algorithmic FLOPs over
    # the active (token, expert) pairs each launch processed; under EP the active
    # pairs of (step, layer) are summed over ranks and spread evenly over the N
    # expert ranks (when the stage's shared-expert GEMM1 rides in the same
    # launch, its 2*R*h*S*e FLOPs are counted too: the bracket then times both)
    h, e = cfg.hidden_dim, cfg.expert_dim
    pair_flops = 4.0 * h * e
    shared_flops = 2.0 * cfg.total_rows / world * h * cfg.num_shared * e
    flops = sum(pair_flops * cnt[ev[2], ev[3], 0] / world
                + (shared_flops if len(ev) > 4 and ev[4] else 0.0) for ev in expert_events)
    merged_launches = sum(1 for ev in expert_events if len(ev) > 4 and ev[4])
    # the event pairs sit inside the captured graph: they hold the last timed replay
    t_exp = sum(ev[0].elapsed_ms(ev[1]) for ev in expert_events) * 1e-3
    n_launch = len(expert_events)
    achieved = flops / t_exp / 1e12
    peak_tf, _, peak_kind = peaks()
    traffic, traffic_src = measured_traffic(args.config)
    device_bytes = int(runner.device_bytes())
    peak_logical = int(res.peak_buffer_bytes)
    pairs = {"active": res.active_pairs, "total": res.total_pairs}

    # e2e through the serving call with host buffers: every step copies its x0 from
    # pinned host memory and its final latent back (single GPU: sample_many, the
    # copies of neighbouring batches overlap the replay; EP: one sample() per step)
    x0_host = torch.as_tensor(x0.values).cpu().pin_memory()
    runner.sample(x0_host)
    barrier()
    if world == 1 and not args.eager:
        out_host = torch.empty_like(x0_host).pin_memory()
        t0 = time.perf_counter()
        runner.sample_many([x0_host] * args.steps, [out_host] * args.steps)
        barrier()
        e2e_s = time.perf_counter() - t0
        final_dice = out_host.clone().numpy().astype(np.float64)
    else:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            runner.sample(x0_host)
        barrier()
        e2e_s = time.perf_counter() - t0
        final_dice = runner._final_host.clone().numpy().astype(np.float64)
    if world > 1:
        e2e_s = float(allreduce([e2e_s], dist.ReduceOp.MAX).item())
    e2e = world * ipg * args.steps / e2e_s
    del runner
    torch.cuda.empty_cache()

    # per-op device time inside the real step (separate timed replay: the events
    # cost a few % of the step, so the headline value above is taken without them)
    breakdown = None
    if world == 1 and not args.no_breakdown:
        breakdown = op_breakdown(D, model, x0, policy, cluster, seed, cfg, args)

    # staleness quality: latent MSE of DICE / interweaved vs the synchronous path
    # (same GPU numerics), and the DICE-vs-synchronous speed ratio on this GPU
    quality = {}
    if not args.no_quality and world == 1:
        finals = {"dice": final_dice}
        for qname, st, pol in (("sync", D.Strategy.SYNCHRONOUS, D.NEUTRAL),
                               ("interweaved", D.Strategy.INTERWEAVED, D.NEUTRAL)):
            r = D.DeviceRunner(model, x0, st, pol, cluster, seed)
            if not args.eager:
                r.capture()
            finals[qname] = r.sample(x0_host).clone().numpy().astype(np.float64)
            if qname == "sync":
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record()
                r.launch()
                ev1.record()
                torch.cuda.synchronize()
                quality["sync_ms_per_run"] = ev0.elapsed_time(ev1)
            del r
            torch.cuda.empty_cache()
        for qname in ("dice", "interweaved"):
            d = finals[qname] - finals["sync"]
            quality[f"{qname}_latent_mse_vs_sync"] = float(np.mean(d * d))
            quality[f"{qname}_rel_l2_vs_sync"] = float(np.linalg.norm(d)
                                                       / np.linalg.norm(finals["sync"]))
        quality["speedup_dice_vs_sync"] = quality["sync_ms_per_run"] / ms_per_step
        quality["policy_of_value"] = conf["policy"]
    elif not args.no_quality and world > 1:
        # the north-star comparison on the same box: the synchronous expert-parallel
        # path (every stage blocks on its dispatch and combine, schedules.py:319-345)
        # timed the same way (device events, max over ranks), and the latent MSE of
        # this run vs it over all ranks' row shards
        from paper_2411_16786_b200.ep import EPRunner
        r = EPRunner(model, x0, D.Strategy.SYNCHRONOUS, D.NEUTRAL, cluster, seed, rank=rank,
                     world=world)
        if not args.eager:
            r.capture()
        final_sync = r.sample(x0_host).clone().numpy().astype(np.float64)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, min(args.steps, 3))
        ev0.record()
        for _ in range(reps):
            r.launch()
        ev1.record()
        barrier()
        r.finish()
        sync_ms = float(allreduce([ev0.elapsed_time(ev1) / reps], dist.ReduceOp.MAX).item())
        d = final_dice - final_sync
        sq = allreduce([float(np.sum(d * d)), float(np.sum(final_sync * final_sync)),
                        float(d.size)], dist.ReduceOp.SUM)
        del r
        torch.cuda.empty_cache()
        quality = {"sync_ep_ms_per_run": sync_ms,
                   "dice_latent_mse_vs_sync": float(sq[0] / sq[2]),
                   "dice_rel_l2_vs_sync": float(np.sqrt(sq[0] / sq[1])),
                   "speedup_dice_vs_sync": sync_ms / ms_per_step,
                   "policy_of_value": conf["policy"],
                   "note": f"synchronous expert parallelism on the same {world} ranks"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_sample(args.config, f"{os.cpu_count()} host threads")
    line = {
        "metric": conf["metric"], "value": value, "unit": "img/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16 GEMM operands / fp32 accum+residual",
        "data": "synthetic (splitmix64 latents, random-init weights)",
        "config": {"workload": conf["workload"], "baseline": conf["baseline"],
                   "images_per_gpu": ipg, "global_batch": ipg * world,
                   "tokens_per_image": cfg.num_tokens, "denoise_steps": cfg.num_steps,
                   "eta": cfg.step_size,
                   "parallelism": (f"ep{world} (experts e//(E/{world}) per GPU, peer-memory "
                                   "all-to-all)") if world > 1 else
                                  f"single-gpu (all {cfg.num_experts} experts)",
                   "l2": "inputs larger than L2: the bf16 weights are streamed every denoising step"},
        "moe_layer_us": ms_per_step * 1e3 / (cfg.num_steps * cfg.num_layers),
        "exposed_a2a_us": exposed_ms * 1e3 / (cfg.num_steps * cfg.num_layers),
        "a2a_parts_us": {k_: v * 1e3 / (cfg.num_steps * cfg.num_layers) for k_, v in (
            ("flag_waits", wait_ms),
            ("main_stream_send_and_regroup_kernels", kern_ms),
            ("waits_for_overlapped_sends", join_ms))},
        # the reference's logical buffer accounting (R*h*2 per occupied slot,
        # schedules.py:185) next to the physical bytes this rank's run holds
        "buffers": {"logical_peak_bytes": peak_logical, "device_bytes": device_bytes},
        "roofline": {"bound": "tensor",
                     "kernel": ("grouped expert FFN (tcgen05 GEMM1+GELU, GEMM2; the stage's "
                                "shared-expert GEMM1 shares the GEMM1 launch)"),
                     "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per grouped-FFN launch pair (ncu --set full)",
                     "traffic_source": traffic_src,
                     "peak_kind": f"{peak_kind} bf16 sustained",
                     "launches": n_launch, "flops_per_pair": pair_flops,
                     "launches_with_shared_gemm1": merged_launches,
                     "share_of_step": t_exp / (ms_per_step / 1e3)},
        "e2e": {"value": e2e, "unit": "img/s",
                "h2d_bytes_per_step": int(x0_host.numel() * 4) * world,
                "d2h_bytes_per_step": int(x0_host.numel() * 4) * world},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "quality": quality,
        "breakdown": breakdown,
        "pairs": pairs,
        "csrc_sha": csrc_digest(),
    }
    if cpu is not None:
        line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(argv, n) -> int:
    """--gpus N outside torchrun: one process per GPU with the torch.distributed
    environment; rank 0 prints the JSON line. Returns the worst exit code."""
    env0 = dict(os.environ)
    env0.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), WORLD_SIZE=str(n),
                LOCAL_WORLD_SIZE=str(n))
    env0.setdefault("NCCL_DEBUG", "INFO")
    procs = []
    for r in range(n):
        env = dict(env0, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *argv], env=env))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="xl256", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-quality", action="store_true")
    ap.add_argument("--no-breakdown", action="store_true")
    ap.add_argument("--eager", action="store_true", help="launch kernels from Python, no CUDA graph")
    ap.add_argument("--overlap", action="store_true",
                    help="run the pending expert FFN on a side stream (intra-GPU interweaving)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if os.environ.get("DICE_BENCH_SAME_DEVICE") != "1":
            import torch
            if torch.cuda.device_count() < args.gpus:
                raise SystemExit(f"bench.py --gpus {args.gpus}: only "
                                 f"{torch.cuda.device_count()} GPU(s) visible")
        return spawn_ranks(sys.argv[1:], args.gpus)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
