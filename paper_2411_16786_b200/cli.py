"""Command-line front end — the GPU counterpart of dicesim's CLI
(/root/reference/pkg/src/dicesim/cli.py).

  python -m paper_2411_16786_b200 run     --config exp.toml [--set model.batch=16] --out DIR
  python -m paper_2411_16786_b200 compare --config exp.toml --out DIR
  python -m paper_2411_16786_b200 sweep   --config exp.toml --out DIR

Reads the reference's TOML experiment schema (schema_version 1: [model] preset
+ field overrides, [cluster], [run] strategy / seed, [policy], [sweep] axes;
--set section.key=value overrides parsed as TOML literals; seed falls back to
DICE_SIM_SEED then 0) and writes reports in the reference's CSV / JSON schema
(metrics.py). Every run executes on the GPU as one captured CUDA graph and its
makespan is the measured device time of a replay. ``validate`` (engine vs the
reference interpreter) is not offered here: that check needs the CPU oracle,
which is test infrastructure (tests/), not part of the package.
Exit codes as the reference: 0 ok, 2 configuration error, 3 numerical divergence.
"""
from __future__ import annotations

import argparse
import dataclasses
import itertools
import math
import os
import sys
import tomllib
from pathlib import Path

from .cluster import ClusterConfig
from .errors import ConfigurationError, ContractError, NumericsError, SimulatorError
from .metrics import build_report, emit, policy_label
from .model import ModelConfig, init_model, preset, sample_x0
from .policies import NEUTRAL, CondStrategy, PolicyConfig, SyncStrategy, dice_policy
from .schedules import DeviceRunner, Strategy

CONFIG_SCHEMA_VERSION = 1
MODEL_FIELDS = {f.name for f in dataclasses.fields(ModelConfig)}
CLUSTER_FIELDS = {f.name for f in dataclasses.fields(ClusterConfig)}
POLICY_FIELDS = {f.name for f in dataclasses.fields(PolicyConfig)}
SWEEP_AXES = ("batch", "num_tokens", "refresh_interval", "period", "warmup", "strategy")


@dataclasses.dataclass(frozen=True)
class Experiment:
    model: ModelConfig
    cluster: ClusterConfig
    strategy: Strategy
    policy: PolicyConfig
    seed: int
    sweep: dict


# ------------------------------------------------------------------ config
def literal(text: str):
    """A --set value as a TOML literal; anything that does not parse is a string."""
    try:
        return tomllib.loads(f"v = {text}")["v"]
    except tomllib.TOMLDecodeError:
        return text


def apply_overrides(config: dict, pairs) -> dict:
    for item in pairs:
        key, eq, raw = item.partition("=")
        if not eq or not key:
            raise ConfigurationError(f"override {item!r} is not KEY=VALUE")
        *path, leaf = key.split(".")
        node = config
        for part in path:
            node = node.setdefault(part, {})
            if not isinstance(node, dict):
                raise ConfigurationError(f"override {item!r} descends into non-table {part!r}")
        node[leaf] = literal(raw)
    return config


def load_config(path, overrides=()) -> dict:
    try:
        with open(path, "rb") as fh:
            config = tomllib.load(fh)
    except tomllib.TOMLDecodeError as exc:
        raise ConfigurationError(f"{path}: invalid TOML: {exc}") from exc
    except OSError as exc:
        raise ConfigurationError(f"{path}: {exc}") from exc
    config = apply_overrides(config, list(overrides))
    version = config.get("schema_version", CONFIG_SCHEMA_VERSION)
    if version != CONFIG_SCHEMA_VERSION:
        raise ConfigurationError(f"unsupported schema_version {version!r}; "
                                 f"this build reads {CONFIG_SCHEMA_VERSION}")
    return config


def _only(section: str, table: dict, allowed) -> None:
    extra = sorted(set(table) - set(allowed))
    if extra:
        raise ConfigurationError(f"[{section}] has unknown keys {extra}; allowed: {sorted(allowed)}")


def _choice(enum_cls, value, field: str):
    try:
        return enum_cls(str(value).lower())
    except ValueError:
        raise ConfigurationError(f"{field} must be one of "
                                 f"{sorted(m.value for m in enum_cls)}, got {value!r}") from None


def model_config(table: dict) -> ModelConfig:
    table = dict(table)
    name = table.pop("preset", None)
    _only("model", table, MODEL_FIELDS)
    try:
        return preset(name, **table) if name is not None else ModelConfig(**table)
    except TypeError as exc:
        raise ConfigurationError(f"[model]: {exc}") from exc


def cluster_config(table: dict) -> ClusterConfig:
    _only("cluster", table, CLUSTER_FIELDS)
    return ClusterConfig(**table)


def policy_config(table: dict) -> PolicyConfig:
    table = dict(table)
    _only("policy", table, POLICY_FIELDS)
    if "sync_strategy" in table:
        table["sync_strategy"] = _choice(SyncStrategy, table["sync_strategy"], "policy.sync_strategy")
    if "cond_strategy" in table:
        table["cond_strategy"] = _choice(CondStrategy, table["cond_strategy"], "policy.cond_strategy")
    if "explicit_layers" in table:
        if not isinstance(table["explicit_layers"], list):
            raise ConfigurationError("policy.explicit_layers must be a list")
        table["explicit_layers"] = frozenset(int(v) for v in table["explicit_layers"])
    if isinstance(table.get("period"), str):
        if table["period"].lower() != "inf":
            raise ConfigurationError(f"policy.period must be a number or \"inf\", "
                                     f"got {table['period']!r}")
        table["period"] = math.inf
    try:
        return PolicyConfig(**table)
    except TypeError as exc:
        raise ConfigurationError(f"[policy]: {exc}") from exc


def resolve_seed(table: dict, env=None) -> int:
    env = os.environ if env is None else env
    if "seed" in table:
        return int(table["seed"])
    raw = env.get("DICE_SIM_SEED")
    if raw is None:
        return 0
    try:
        return int(raw)
    except ValueError:
        raise ConfigurationError(f"DICE_SIM_SEED must be an integer, got {raw!r}") from None


def build_experiment(config: dict) -> Experiment:
    _only("<top level>", config, {"schema_version", "model", "cluster", "run", "policy", "sweep"})
    run = dict(config.get("run", {}))
    _only("run", run, {"strategy", "seed"})
    sweep = dict(config.get("sweep", {}))
    _only("sweep", sweep, SWEEP_AXES)
    for axis, values in sweep.items():
        if not isinstance(values, list) or not values:
            raise ConfigurationError(f"sweep.{axis} must be a non-empty list")
    return Experiment(model=model_config(config.get("model", {})),
                      cluster=cluster_config(config.get("cluster", {})),
                      strategy=_choice(Strategy, run.get("strategy", "synchronous"), "run.strategy"),
                      policy=policy_config(config.get("policy", {})),
                      seed=resolve_seed(run), sweep=sweep)


def sweep_points(exp: Experiment) -> list:
    """Cross product of the sweep axes: axes in name order, values in configured
    order, the last axis fastest (the reference's expand_sweep order)."""
    axes = sorted(exp.sweep)
    if not axes:
        return [exp]
    points = []
    for combo in itertools.product(*(exp.sweep[a] for a in axes)):
        model, policy, strategy = exp.model, exp.policy, exp.strategy
        for axis, value in zip(axes, combo):
            if axis in ("batch", "num_tokens"):
                model = dataclasses.replace(model, **{axis: int(value)})
            elif axis == "strategy":
                strategy = _choice(Strategy, value, "sweep.strategy")
            elif axis == "period":
                policy = dataclasses.replace(policy, period=math.inf if value == "inf"
                                             else float(value))
            else:
                policy = dataclasses.replace(policy, **{axis: int(value)})
        points.append(dataclasses.replace(exp, model=model, policy=policy, strategy=strategy,
                                          sweep={}))
    return points


# --------------------------------------------------------------- execution
def timed_run(model, x0, strategy, policy, cluster, seed, timeline_path=None):
    """One run on the GPU: captured as a CUDA graph, warmed, then one timed
    replay (CUDA events) whose device time is the run's makespan."""
    import torch
    runner = DeviceRunner(model, x0, strategy, policy, cluster, seed)
    runner.capture()
    runner.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    runner.launch()
    e1.record()
    torch.cuda.synchronize()
    result = runner.finish(gpu_seconds=e0.elapsed_time(e1) * 1e-3)
    if timeline_path is not None:
        traced = DeviceRunner(model, x0, strategy, policy, cluster, seed, timeline=True)
        tl = traced.run().timeline
        Path(timeline_path).write_text(tl.to_json() + "\n")
    return result


def execute(exp: Experiment, timeline_dir=None, tag=""):
    model = init_model(exp.model, seed=exp.seed)
    x0 = sample_x0(exp.model, seed=exp.seed)
    baseline = timed_run(model, x0, Strategy.SYNCHRONOUS, NEUTRAL, exp.cluster, exp.seed)
    if exp.strategy is Strategy.SYNCHRONOUS and exp.policy == NEUTRAL:
        result = baseline
    else:
        name = f"timeline_{tag}.json" if tag else "timeline.json"
        result = timed_run(model, x0, exp.strategy, exp.policy, exp.cluster, exp.seed,
                           None if timeline_dir is None else Path(timeline_dir) / name)
    return build_report(result, baseline)


def write_reports(reports, out_dir, name, fmt) -> Path:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    path = out / f"{name}.{fmt}"
    emit(reports, fmt, path)
    return path


def summarize(reports, stream=None) -> None:
    stream = sys.stdout if stream is None else stream
    print(f"{'strategy':<12} {'policy':<44} {'divergence':>12} {'makespan_s':>12} "
          f"{'speedup':>8}", file=stream)
    for r in reports:
        print(f"{r.strategy:<12} {r.policy:<44} {r.divergence:>12.3e} "
              f"{r.makespan_seconds:>12.6f} {r.speedup_vs_sync:>8.3f}", file=stream)


COMPARE_VARIANTS = (
    (Strategy.SYNCHRONOUS, NEUTRAL, "synchronous"),
    (Strategy.DISPLACED, NEUTRAL, "displaced"),
    (Strategy.INTERWEAVED, NEUTRAL, "interweaved"),
    (Strategy.INTERWEAVED, dice_policy(), "dice"),
)


def cmd_run(args) -> int:
    exp = build_experiment(load_config(args.config, args.set))
    report = execute(exp, timeline_dir=args.out if args.timeline else None)
    path = write_reports([report], args.out, "report", args.format)
    summarize([report])
    print(f"wrote {path}", file=sys.stderr)
    return 0


def cmd_compare(args) -> int:
    exp = build_experiment(load_config(args.config, args.set))
    reports = [execute(dataclasses.replace(exp, strategy=s, policy=p),
                       timeline_dir=args.out if args.timeline else None, tag=tag)
               for s, p, tag in COMPARE_VARIANTS]
    path = write_reports(reports, args.out, "compare", args.format)
    summarize(reports)
    print(f"wrote {path}", file=sys.stderr)
    return 0


def cmd_sweep(args) -> int:
    exp = build_experiment(load_config(args.config, args.set))
    reports = [execute(pt, timeline_dir=args.out if args.timeline else None, tag=f"{i:03d}")
               for i, pt in enumerate(sweep_points(exp))]
    path = write_reports(reports, args.out, "sweep", args.format)
    summarize(reports)
    print(f"wrote {path} ({len(reports)} rows)", file=sys.stderr)
    return 0


def make_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="python -m paper_2411_16786_b200",
        description="DICE expert-parallel MoE-DiT sampling on B200: run, compare and sweep "
                    "experiments from the reference's TOML configs.")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, text in (("run", "run one experiment against its synchronous baseline"),
                       ("compare", "synchronous / displaced / interweaved / DICE on one model"),
                       ("sweep", "cross product over the [sweep] axes")):
        p = sub.add_parser(name, help=text)
        p.add_argument("--config", required=True, help="TOML experiment config")
        p.add_argument("--set", action="append", default=[], metavar="KEY=VALUE",
                       help="override a config entry (repeatable), e.g. --set model.batch=16")
        p.add_argument("--out", default=".", metavar="DIR", help="report directory")
        p.add_argument("--format", choices=("csv", "json"), default="csv")
        p.add_argument("--timeline", action="store_true",
                       help="also export the measured per-stage timeline JSON")
    return parser


def main(argv=None) -> int:
    args = make_parser().parse_args(argv)
    handler = {"run": cmd_run, "compare": cmd_compare, "sweep": cmd_sweep}[args.command]
    try:
        return handler(args)
    except NumericsError as exc:
        step = getattr(exc, "step", None)
        print(f"numerical divergence{'' if step is None else f' at step {step}'}: {exc}",
              file=sys.stderr)
        return 3
    except (ConfigurationError, ContractError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except SimulatorError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
