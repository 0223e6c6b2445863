"""Expert placement and all-to-all byte accounting — drop-in for the
placement half of dicesim.cluster (/root/reference/pkg/src/dicesim/cluster.py).

The alpha-beta SimTimeline (cluster.py:112-216) is a simulated wire; on B200
the wire is real (NCCL / NVLink) and time is measured with CUDA events, so the
timeline is not restated. ClusterConfig keeps the reference fields for API
parity; only num_devices and bytes_per_element affect results.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ConfigurationError, ContractError
from .model import RouteDecision

DEFAULT_ALPHA = 0.0
DEFAULT_BETA = 1.3289168938023188e-07
DEFAULT_COMPUTE_RATE = 1.0e9
DEFAULT_OP_OVERHEAD = 31403
DEFAULT_NUM_DEVICES = 8


@dataclass(frozen=True)
class ClusterConfig:
    """Same fields and validation as cluster.py:28-50."""
    num_devices: int = DEFAULT_NUM_DEVICES
    alpha: float = DEFAULT_ALPHA
    beta: float = DEFAULT_BETA
    bytes_per_element: int = 2
    compute_rate: float = DEFAULT_COMPUTE_RATE
    op_overhead_elements: int = DEFAULT_OP_OVERHEAD

    def __post_init__(self):
        if self.num_devices < 1:
            raise ConfigurationError(f"num_devices must be >= 1, got {self.num_devices}")
        if self.alpha < 0 or self.beta < 0:
            raise ConfigurationError("alpha and beta must be >= 0")
        if self.bytes_per_element < 1:
            raise ConfigurationError("bytes_per_element must be >= 1")
        if not self.compute_rate > 0:
            raise ConfigurationError("compute_rate must be > 0")
        if self.op_overhead_elements < 0:
            raise ConfigurationError("op_overhead_elements must be >= 0")


@dataclass(frozen=True)
class Placement:
    expert_device: torch.Tensor   # [num_experts] int64
    token_home: torch.Tensor      # [rows] int64
    num_devices: int


def build_placement(num_experts: int, num_devices: int, num_rows: int, device="cpu") -> Placement:
    """Contiguous expert blocks, near-even contiguous token shards (cluster.py:61-72)."""
    if num_devices < 1:
        raise ConfigurationError(f"num_devices must be >= 1, got {num_devices}")
    if num_experts % num_devices != 0:
        raise ConfigurationError(
            f"num_experts={num_experts} not divisible by num_devices={num_devices}")
    per = num_experts // num_devices
    expert_device = torch.arange(num_experts, device=device) // per
    token_home = (torch.arange(num_rows, device=device) * num_devices) // num_rows
    return Placement(expert_device=expert_device, token_home=token_home, num_devices=num_devices)


def shard_rows(num_rows: int, num_devices: int, rank: int) -> tuple:
    """[first, last) global rows homed on `rank` under token_home = (t*D)//R."""
    first = -(-rank * num_rows // num_devices)
    last = -(-(rank + 1) * num_rows // num_devices)
    return first, last


def _pair_devices(route: RouteDecision, placement: Placement):
    ids = route.expert_ids.to(placement.expert_device.device).long()
    src = placement.token_home[:, None].expand_as(ids)
    dst = placement.expert_device[ids]
    return src, dst


def plan_all_to_all(route: RouteDecision, placement: Placement, active, hidden_dim: int,
                    bytes_per_element: int) -> int:
    """On-wire bytes of one direction: remote active pairs only (cluster.py:82-90)."""
    src, dst = _pair_devices(route, placement)
    remote = src != dst
    if active is not None:
        remote = remote & torch.as_tensor(active, device=remote.device).bool()
    return int(remote.sum().item()) * hidden_dim * bytes_per_element


def per_device_bytes(route: RouteDecision, placement: Placement, active, hidden_dim: int,
                     bytes_per_element: int, direction: str) -> torch.Tensor:
    """Bytes each device puts on the wire (cluster.py:93-109)."""
    if direction not in ("dispatch", "combine"):
        raise ContractError(f"direction must be dispatch or combine, got {direction!r}")
    src, dst = _pair_devices(route, placement)
    remote = src != dst
    if active is not None:
        remote = remote & torch.as_tensor(active, device=remote.device).bool()
    origin = src if direction == "dispatch" else dst
    counts = torch.bincount(origin[remote].reshape(-1), minlength=placement.num_devices)
    return counts * hidden_dim * bytes_per_element
