"""gloo worker for the CPU expert-parallel protocol test: runs EPRunner's real
host control flow and handle exchange (torch.distributed gloo) with the device
calls stubbed, and records every flag operation and window data access."""
import json
import os
import pickle
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2411_16786_b200 as D  # noqa: E402
from paper_2411_16786_b200 import _lib, ep, ops, policies  # noqa: E402

FAKE_BASE = 1 << 40


class FakeWindow(ep.Window):
    def __init__(self, L, Dn, cap, k, nmax, hp, device):
        self._layout(L, Dn, cap, k, nmax, hp)
        self.ptr = FAKE_BASE * (dist.get_rank() + 1)

    def view(self, offset, shape, dtype):
        return torch.zeros(shape, dtype=dtype)

    def handle(self):
        return b"FAKE" + bytes([dist.get_rank() + 1]) + b"x" * 59

    def free(self):
        pass


def fake_call(name, *args):
    if name == "dice_ipc_open":
        rank = args[0].value[4] - 1
        args[1]._obj.value = FAKE_BASE * (rank + 1)
    return 0


class FakeOps:
    EPI_STORE_BF16, EPI_GELU_BF16, EPI_STORE_F32, EPI_GELU_RESID = range(4)
    pad64 = staticmethod(ops.pad64)
    pad_hidden = staticmethod(ops.pad_hidden)
    COND_CODES = ops.COND_CODES

    @staticmethod
    def _stream():
        return 0

    @staticmethod
    def permute_max_rows(n, k, E):
        return ((n * k + 255 * E + 255) // 256) * 256

    @staticmethod
    def permute_scratch_ints(n, k, E):
        return max(1, (n * k + 1023) // 1024) * E

    class DeviceEvent:
        def record(self):
            pass

        def elapsed_ms(self, other):
            return 0.0

    def __getattr__(self, name):
        return lambda *a, **k: None


def cpu_model(cfg, experts):
    hp, ep_ = ops.pad_hidden(cfg.hidden_dim), ops.pad64(cfg.expert_dim)
    El = experts[1] - experts[0]
    S = cfg.num_shared
    bf = torch.bfloat16
    layers = [D.model.LayerWeights(torch.zeros(hp, hp, dtype=bf), torch.zeros(cfg.num_experts, hp),
                                   torch.zeros(El * ep_, hp, dtype=bf), torch.zeros(El * hp, ep_, dtype=bf),
                                   torch.zeros(S * ep_, hp, dtype=bf) if S else None,
                                   torch.zeros(hp, S * ep_, dtype=bf) if S else None)
              for _ in range(cfg.num_layers)]
    return D.ToyModel(config=cfg, seed=0, layers=layers, experts=experts, hp=hp, ep=ep_, device="cpu")


def main(a):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{a['port']}", rank=a["rank"],
                            world_size=a["world"])
    ep.Window = FakeWindow
    _lib.call = fake_call
    fake = FakeOps()
    ep.ops = fake
    policies.ops = fake
    rank, world = a["rank"], a["world"]
    cfg = D.ModelConfig(**a["cfg"])
    El = cfg.num_experts // world
    pol = {"neutral": D.NEUTRAL, "dice": D.dice_policy(refresh_interval=2, warmup=2, period=3),
           "deep": D.PolicyConfig(sync_strategy=D.SyncStrategy.DEEP)}[a["policy"]]
    a0, a1 = D.cluster.shard_rows(cfg.total_rows, world, rank)
    x0 = D.ActivationBlock(torch.zeros(a1 - a0, cfg.hidden_dim), 0)
    r = ep.EPRunner(cpu_model(cfg, (rank * El, (rank + 1) * El)), x0, D.Strategy(a["strategy"]),
                    pol, D.ClusterConfig(num_devices=world), 3, rank=rank, world=world)
    trace = []
    r.grp.trace = trace
    for _ in range(a.get("runs", 1)):
        r._reset_state()
        for step in range(cfg.num_steps):
            r._run_step(step)
        r._drain()
    w = r.win
    layout = dict(o_rx_ready=w.o_rx_ready, o_cx_ready=w.o_cx_ready, o_rx_free=w.o_rx_free,
                  o_cx_free=w.o_cx_free, L=w.L, D=w.D)
    logs = [None] * world
    dist.all_gather_object(logs, dict(rank=rank, base=r.grp.base, trace=trace, layout=layout,
                                      records=[(s.layer, s.used_step, s.generated_step)
                                               for s in r.records]))
    if rank == 0:
        with open(a["out"], "wb") as f:
            pickle.dump(logs, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(json.loads(sys.argv[1]))
