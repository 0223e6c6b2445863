"""CPU, world_size 2 and 4 over gloo: the expert-parallel exchange protocol
(EPRunner host control flow, IPC-handle rendezvous through torch.distributed,
ready/free flag handshakes) is simulated under many random interleavings of
the ranks' stream operations (each rank's main stream and, for the
interweaved schedule, its comm stream carrying the overlapped dispatch sends,
joined only by event records / waits). Checks: no deadlock; every receive region is
written exactly once before it is read and read before it is rewritten; every
consume of a home's pair rows finds, from every expert rank, the combine of
exactly the step it consumes (stored and signalled; never a newer one) — no
data race; every flag returns to its initial value (graph-replay safe); all
ranks follow the reference staleness law."""
import json
import os
import pickle
import random
import socket
import subprocess
import sys
import tempfile

import pytest

from oracle import dice_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
FAKE_BASE = 1 << 40

CFG = dict(num_layers=3, num_experts=8, num_shared=1, top_k=2, hidden_dim=8, expert_dim=16,
           num_tokens=4, batch=2, num_steps=7, step_size=1e-3)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def collect(world, strategy, policy, runs=1):
    port = free_port()
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "logs.pkl")
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "ep_protocol_worker.py"),
                                   json.dumps(dict(rank=r, world=world, port=port, cfg=CFG,
                                                   strategy=strategy, policy=policy, out=out,
                                                   runs=runs))])
                 for r in range(world)]
        for p in procs:
            p.wait(timeout=180)
            assert p.returncode == 0
        with open(out, "rb") as f:
            return pickle.load(f)


def initial_flags(logs):
    flags = {}
    for lg in logs:
        lay, b = lg["layout"], FAKE_BASE * (lg["rank"] + 1)
        n = lay["L"] * lay["D"]
        for key, init in (("o_rx_ready", 0), ("o_cx_ready", 0), ("o_rx_free", 1), ("o_cx_free", 0)):
            for i in range(n):
                flags[b + lay[key] + 4 * i] = init
    return flags


def simulate(logs, seed):
    """Random interleaving of every (rank, stream) op queue: a rank's main
    stream and its comm stream (overlapped dispatch sends) run concurrently,
    ordered only by their event records / waits."""
    rng = random.Random(seed)
    flags = initial_flags(logs)
    init = dict(flags)
    full = set()            # receive regions holding unread data
    cx = {}                 # pair-row region -> (step of its combine, signalled)
    queues = {}
    for r, lg in enumerate(logs):
        for op in lg["trace"]:
            queues.setdefault((r, op[3]), []).append(op)
    pcs = {q: 0 for q in queues}
    recorded = set()        # (rank, event id)
    ureads = set()          # (rank, send number) whose u16 read has executed
    steps = 0
    while True:
        ready = []
        for q, tr in queues.items():
            if pcs[q] >= len(tr):
                continue
            op = tr[pcs[q]]
            if op[0] == "wait" and not all(flags[a] == op[2] for a in op[1]):
                continue
            if op[0] == "wait_event" and (q[0], op[2]) not in recorded:
                continue
            ready.append(q)
        if not ready:
            break
        q = rng.choice(ready)
        r = q[0]
        op = queues[q][pcs[q]]
        if op[0] == "record":
            recorded.add((r, op[2]))
        elif op[0] == "write":                    # flag write (stream memop)
            for a in op[1]:
                assert a in flags, hex(a)
                flags[a] = op[2]
        elif op[0] == "kwrite":                   # kernel stores into window regions
            for reg in map(tuple, op[1]):
                if reg[0] == "cx":                # pair rows: the combine of step op[2]
                    cx[reg] = (op[2], False)
                    continue
                assert reg not in full, f"rank {r} overwrites unread {reg}"
                full.add(reg)
        elif op[0] == "read":                     # kernel reads receive regions
            for reg in map(tuple, op[1]):
                assert reg in full, f"rank {r} reads {reg} before it was written"
                full.discard(reg)
        elif op[0] == "arrive":                   # home: combine stores signalled
            for reg in map(tuple, op[1]):
                assert reg in cx and not cx[reg][1], f"rank {r}: {reg} arrives without a store"
                cx[reg] = (cx[reg][0], True)
        elif op[0] == "uread":                    # a send kernel read u16 / its payload
            ureads.add((r, op[2]))
        elif op[0] == "uwrite":                   # local_block overwrites u16
            assert op[2] == 0 or (r, op[2]) in ureads, \
                f"rank {r}: u16 overwritten before send {op[2]} read it"
        elif op[0] == "consume":                  # home reads its pair rows
            for reg in map(tuple, op[1]):
                got = cx.get(reg)
                assert got == (op[2], True), f"rank {r} consumes {reg}: has {got}, wants step {op[2]}"
        pcs[q] += 1
        steps += 1
    done = all(pcs[q] >= len(t) for q, t in queues.items())
    assert done, f"deadlock: pcs={pcs}"
    assert not full, f"unread regions at the end: {sorted(full)[:4]}"
    assert all(arrived for _, arrived in cx.values())
    assert flags == init, "flags not restored"
    return steps


@pytest.mark.parametrize("world,strategy,policy", [(2, "synchronous", "neutral"),
                                                   (2, "interweaved", "dice"),
                                                   (4, "interweaved", "neutral"),
                                                   (4, "interweaved", "deep"),
                                                   (2, "displaced", "neutral"),
                                                   (2, "displaced", "dice"),
                                                   (4, "displaced", "deep")])
def test_exchange_protocol_random_interleavings(world, strategy, policy):
    logs = collect(world, strategy, policy, runs=2)
    # the trace records kernel writes as ("write", [regions]) only when the
    # items are region tuples; split them from flag writes (ints)
    for lg in logs:
        fixed = []
        for op in lg["trace"]:
            if op[0] == "write" and op[1] and not isinstance(op[1][0], int):
                fixed.append(("kwrite", op[1], op[2], op[3]))
            else:
                fixed.append(op)
        lg["trace"] = fixed
    recs = [lg["records"] for lg in logs]
    assert all(r == recs[0] for r in recs), "ranks disagree on the schedule"
    # ... and the schedule is the reference's (the oracle's staleness records;
    # of the last of two runs back to back)
    g = O.Geometry(**CFG)
    pol = {"neutral": O.Policy(), "dice": O.dice_defaults(refresh_interval=2, warmup=2, period=3),
           "deep": O.Policy(sync_strategy=O.SYNC_DEEP)}[policy]
    ref = O.run_schedule(g, O.init_params(g, 3), O.initial_latent(g, 3), strategy, pol, world, 3)
    assert recs[0] == [tuple(t) for t in ref.staleness]
    if strategy == "interweaved":   # the overlapped dispatch really uses the comm stream
        assert any(op[3] == "comm" for lg in logs for op in lg["trace"])
    for seed in range(40):
        simulate(logs, seed)


def test_handles_exchanged_over_gloo():
    logs = collect(2, "synchronous", "neutral")
    for lg in logs:
        assert lg["base"] == [FAKE_BASE * (r + 1) for r in range(2)]
