"""Expert-parallel DICE sampling across GPUs (one process per GPU).

Placement follows the reference (cluster.py:61-72): routed expert e lives on
rank e // (E/D); token row t is homed on rank (t*D)//R. W_mix, W_gate and the
shared experts are replicated (row-wise data parallel work).

Exchange: every rank cudaMallocs one window allocation, exports it with CUDA
IPC and maps every peer's (handles travel through torch.distributed object
collectives; that is the only use of the process group on the data path's
setup). The dispatch kernel stores each active pair's bf16 row straight into
the expert rank's window; the expert rank's GEMM2 epilogue stores each
output row, with its gate and expert id, straight into the home rank's pair
rows — which live in the home's window and ARE its token cache rows / combine
slot (see DeviceRunner), so the combine needs no kernel at the home.
Completion uses constant-valued flags (ready / free per layer and peer)
driven by batched stream memory operations, so the schedule keeps
host-deterministic control flow and a whole run captures into one CUDA graph
per rank.

Schedule (schedules.py:372-402, PAPER §4.1): dispatch(l) is sent in stage l and
expert-processed in stage l+1 (or at a flush); its combine arrival is awaited
at the start of stage l of the next step, right before decide(l) so the
TokenCache sees the reference's decide/assemble order (policies.py:159-208),
and consumed with one-step staleness; once the consume has read the layer's
pair rows, the home frees them for the next combine. Selective-sync / warmup
/ periodic stages run the blocking dispatch -> experts -> combine sequence.
"""
from __future__ import annotations

import ctypes
import dataclasses
import hashlib
import os

import numpy as np
import torch

from . import _lib, ops
from .cluster import ClusterConfig, shard_rows
from .errors import ConfigurationError, ContractError, NumericalDivergenceError
from .model import ActivationBlock, RouteDecision, ToyModel, model_hash, mix64, _X0_STREAM_TAG
from .policies import CondStrategy, PolicyConfig, TokenCache, is_sync_step, select_sync_layers
from .schedules import INT32_MAX, RunResult, StalenessRecord, Strategy


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (for torch.as_tensor)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


_TYPESTR = {torch.float32: "<f4", torch.bfloat16: "<V2", torch.int32: "<i4", torch.uint8: "|u1",
            torch.int64: "<i8"}


class Window:
    """One cudaMalloc'd allocation: receive windows, the rank's pair rows /
    gates / ids (written by the expert ranks) and flags. Every rank uses the
    same layout (sized by the largest shard, nmax rows), so peers compute
    addresses from the base pointer alone."""

    def __init__(self, L, D, cap, k, nmax, hp, device):
        self._layout(L, D, cap, k, nmax, hp)
        h = ctypes.c_void_p()
        torch.cuda.set_device(device)
        _lib.call("dice_device_alloc", self.nbytes, ctypes.byref(h))
        self.ptr = int(h.value)
        # receive regions start free (rx_free = 1); pair rows are freed by their
        # home right before each expert call of the layer (cx_free starts at 0)
        self.view(self.o_rx_free, (L * D,), torch.int32).fill_(1)
        torch.cuda.synchronize()

    def _layout(self, L, D, cap, k, nmax, hp):
        self.L, self.D, self.cap, self.k, self.nmax, self.hp = L, D, cap, k, nmax, hp
        off = 0

        def take(nbytes):
            nonlocal off
            start = off
            off += (nbytes + 255) // 256 * 256
            return start

        self.o_rx_rows = take(L * D * cap * hp * 2)
        self.o_rx_meta = take(L * D * cap * 16)
        self.o_rx_count = take(L * D * 4)
        self.row_block = k * nmax * hp * 2        # bytes of one layer's pair rows
        self.o_cx_rows = take(L * self.row_block)
        self.o_cx_gates = take(L * nmax * k * 4)
        self.o_cx_ids = take(L * nmax * k * 4)
        self.o_rx_ready = take(L * D * 4)
        self.o_cx_ready = take(L * D * 4)
        self.o_rx_free = take(L * D * 4)
        self.o_cx_free = take(L * D * 4)
        self.nbytes = off

    def pair_views(self, n):
        """This rank's pair rows bf16 [L, k, n, hp], gates f32 [L, n, k], ids
        int32 [L, n, k] (layer blocks sized for nmax rows)."""
        L, k, hp, nmax = self.L, self.k, self.hp, self.nmax
        flat = self.view(self.o_cx_rows, (L * k * nmax * hp,), torch.bfloat16)
        rows = torch.as_strided(flat, (L, k, n, hp), (k * nmax * hp, n * hp, hp, 1))
        g = self.view(self.o_cx_gates, (L * nmax * k,), torch.float32)
        gates = torch.as_strided(g, (L, n, k), (nmax * k, k, 1))
        i = self.view(self.o_cx_ids, (L * nmax * k,), torch.int32)
        ids = torch.as_strided(i, (L, n, k), (nmax * k, k, 1))
        return rows, gates, ids

    def view(self, offset, shape, dtype):
        if dtype is torch.bfloat16:
            t = torch.as_tensor(_CudaArray(self.ptr + offset, shape, "<i2"), device="cuda")
            return t.view(torch.bfloat16)
        return torch.as_tensor(_CudaArray(self.ptr + offset, shape, _TYPESTR[dtype]), device="cuda")

    def handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _lib.call("dice_ipc_get_handle", ctypes.c_void_p(self.ptr), buf)
        return buf.raw

    def free(self):
        if self.ptr:
            _lib.load().dice_device_free(ctypes.c_void_p(self.ptr))
            self.ptr = 0


def _u64_array(values):
    arr = (ctypes.c_uint64 * max(1, len(values)))(*[int(v) for v in values])
    return arr


class EPGroup:
    """Rank-local view of the D windows (own + IPC-mapped peers)."""

    def __init__(self, window: Window, rank: int, world: int, pg=None):
        import torch.distributed as dist
        self.win, self.rank, self.world = window, rank, world
        handles = [None] * world
        if world > 1:
            dist.all_gather_object(handles, window.handle(), group=pg)
        self.base = []
        self._opened = []
        for r in range(world):
            if r == rank:
                self.base.append(window.ptr)
            else:
                h = ctypes.c_void_p()
                _lib.call("dice_ipc_open", ctypes.c_char_p(handles[r]), ctypes.byref(h))
                self.base.append(int(h.value))
                self._opened.append(int(h.value))

    def close(self):
        for p in self._opened:
            _lib.load().dice_ipc_close(ctypes.c_void_p(p))
        self._opened = []

    # addresses -----------------------------------------------------------
    def rx_rows(self, owner, layer, src):
        w = self.win
        return self.base[owner] + w.o_rx_rows + ((layer * w.D + src) * w.cap) * w.hp * 2

    def rx_meta(self, owner, layer, src):
        w = self.win
        return self.base[owner] + w.o_rx_meta + ((layer * w.D + src) * w.cap) * 16

    def rx_count(self, owner, layer, src):
        w = self.win
        return self.base[owner] + w.o_rx_count + (layer * w.D + src) * 4

    def cx_rows(self, owner, layer):
        w = self.win
        return self.base[owner] + w.o_cx_rows + layer * w.row_block

    def cx_gates(self, owner, layer):
        w = self.win
        return self.base[owner] + w.o_cx_gates + layer * w.nmax * w.k * 4

    def cx_ids(self, owner, layer):
        w = self.win
        return self.base[owner] + w.o_cx_ids + layer * w.nmax * w.k * 4

    def flag(self, kind, owner, layer, peer):
        w = self.win
        o = {"rx_ready": w.o_rx_ready, "cx_ready": w.o_cx_ready, "rx_free": w.o_rx_free,
             "cx_free": w.o_cx_free}[kind]
        return self.base[owner] + o + (layer * w.D + peer) * 4

    # stream memops ---------------------------------------------------------
    trace = None   # optional list: the protocol simulation test records every op
    stream = "main"   # the rank's stream the next ops are issued on (trace tag)

    def stream_op(self, kind, stream, event_id):
        """Record an event record / wait between the rank's two streams (test tracing)."""
        if self.trace is not None:
            self.trace.append((kind, stream, event_id, stream))

    def wait(self, addrs, value):
        if self.trace is not None:
            self.trace.append(("wait", [int(a) for a in addrs], value, self.stream))
        arr = _u64_array(addrs)
        _lib.call("dice_stream_wait_eq", arr, len(addrs), value, ops._stream())

    def write(self, addrs, value):
        if self.trace is not None:
            self.trace.append(("write", [int(a) for a in addrs], value, self.stream))
        arr = _u64_array(addrs)
        _lib.call("dice_stream_write", arr, len(addrs), value, ops._stream())

    def data(self, kind, regions, gen=None):
        """Record a data access of a kernel (test tracing only); gen: the step
        whose combine a pair-row store writes / a consume expects."""
        if self.trace is not None:
            self.trace.append((kind, regions, gen, self.stream))


class _EPPayload:
    def __init__(self, n, k, device):
        self.ids = torch.zeros(n, k, dtype=torch.int32, device=device)
        self.gates = torch.zeros(n, k, dtype=torch.float32, device=device)
        self.active = torch.ones(n, k, dtype=torch.uint8, device=device)
        self.write = torch.zeros(n, k, dtype=torch.uint8, device=device)
        self.layer = -1
        self.gen = -1


def sample_x0_shard(config, seed: int, rows: tuple, device="cuda") -> ActivationBlock:
    """Rows [r0, r1) of sample_x0 (model.py:181-186): the tagged stream at offset r0*h."""
    r0, r1 = rows
    x = torch.empty(r1 - r0, config.hidden_dim, dtype=torch.float32, device=device)
    ops.splitmix_fill(x, mix64(seed ^ _X0_STREAM_TAG), r0 * config.hidden_dim, r1 - r0,
                      config.hidden_dim, 1.0)
    return ActivationBlock(values=x, generated_step=0)


class EPRunner:
    """One rank of an expert-parallel sampling run (ScheduleRunner semantics,
    schedules.py:142-490: SYNCHRONOUS, DISPLACED and INTERWEAVED).

    DISPLACED (schedules.py:347-370) keeps each layer's dispatch in the peers'
    receive windows for a whole step: stage (s, l) consumes the layer's pair
    rows (step s-2's combine, staleness 2), then expert-processes the dispatch
    of step s-1 (its combine arrival is awaited at the start of stage (s+1, l),
    still after decide(s) as in the reference), then sends the new one into the
    windows that processing just freed, so one window per layer suffices. A dispatch a sync stage supersedes is drained unprocessed (the reference
    drops it, its bytes stay counted), and a sync stage's own dispatch, which
    the reference re-processes at the next stage, is already in the slot
    (every pair of a forced refresh is active, so re-assembling it changes
    nothing): only its combine bytes are counted again."""

    def __init__(self, model: ToyModel, x0_shard: ActivationBlock, strategy: Strategy,
                 policy: PolicyConfig, cluster: ClusterConfig, seed: int, *, rank: int,
                 world: int, pg=None, time_waits: bool = False, time_experts: bool = False,
                 overlap_dispatch: bool = True):
        """overlap_dispatch: in asynchronous interweaved stages the dispatch
        send (decide state ready -> group by destination -> P2P row stores ->
        ready flags) runs on a second stream, overlapping the stage's expert
        FFN and consume; the main stream joins it before the next local_block
        GEMM overwrites the rows it reads (and the join's wait is counted as
        exposed all-to-all time)."""
        cfg = model.config
        if cluster.num_devices != world:
            raise ConfigurationError(f"cluster.num_devices={cluster.num_devices} != world={world}")
        if cfg.num_experts % world:
            raise ConfigurationError(f"num_experts={cfg.num_experts} not divisible by {world}")
        if world > 16:
            raise ConfigurationError("up to 16 ranks")
        El = cfg.num_experts // world
        if model.experts != (rank * El, (rank + 1) * El):
            raise ContractError(f"rank {rank} must hold experts [{rank * El}, {(rank + 1) * El})")
        self.r0, self.r1 = shard_rows(cfg.total_rows, world, rank)
        n = self.r1 - self.r0
        if tuple(x0_shard.values.shape) != (n, cfg.hidden_dim) or x0_shard.generated_step != 0:
            raise ContractError(f"rank {rank} x0 shard must be [{n}, {cfg.hidden_dim}] at step 0")
        if policy.cond_strategy is CondStrategy.RANDOM and policy.cond_seed is None:
            policy = dataclasses.replace(policy, cond_seed=seed)
        self.model, self.cfg, self.x0 = model, cfg, x0_shard
        self.strategy, self.policy, self.cluster, self.seed = strategy, policy, cluster, seed
        self.rank, self.world, self.pg, self.El = rank, world, pg, El
        self.time_waits = time_waits
        self.time_experts = time_experts
        dev = model.device
        self.dev = dev
        self.cuda = str(dev).startswith("cuda")
        self.overlap_dispatch = (overlap_dispatch and strategy is Strategy.INTERWEAVED
                                 and world > 1)
        self.comm = torch.cuda.Stream(device=dev) if self.overlap_dispatch and self.cuda else None
        self._comm_pending = None       # event of the last send issued on the comm stream
        self._uread = 0                 # sends issued (test tracing of the u16 reuse)
        self._ev_id = 0
        k, E, S, hp, ep = cfg.top_k, cfg.num_experts, cfg.num_shared, model.hp, model.ep
        self.n, self.k, self.E, self.S, self.hp, self.ep = n, k, E, S, hp, ep
        self.shard_n = [shard_rows(cfg.total_rows, world, r)[1] - shard_rows(cfg.total_rows, world, r)[0]
                        for r in range(world)]
        n_max = max(self.shard_n)
        self.cap = n_max * k
        L = cfg.num_layers
        self.win = Window(L, world, self.cap, k, n_max, hp,
                          torch.cuda.current_device() if str(dev).startswith("cuda") else None)
        self.grp = EPGroup(self.win, rank, world, pg)
        f32, bf = torch.float32, torch.bfloat16
        self.x32 = torch.zeros(n, hp, dtype=f32, device=dev)
        self.x16 = torch.zeros(n, hp, dtype=bf, device=dev)
        self.h32 = torch.zeros(n, hp, dtype=f32, device=dev)
        self.h16 = torch.zeros(n, hp, dtype=bf, device=dev)
        self.u32 = torch.zeros(n, hp, dtype=f32, device=dev)
        self.u16 = torch.zeros(n, hp, dtype=bf, device=dev)
        # the shared-expert GEMM1 rides in the expert GEMM1 launch (see DeviceRunner)
        self.merge_gemm1 = cfg.num_shared > 0
        total = world * self.cap
        self.max_rows = ops.permute_max_rows(total, 1, El)
        self.hbuf = torch.empty(self.max_rows, ep, dtype=bf, device=dev)
        self.x_perm = torch.empty(self.max_rows, hp, dtype=bf, device=dev)
        # permuted row -> window entry: the expert GEMM2 epilogue stores each finished
        # row straight into its home rank's pair rows (fused combine all-to-all)
        self.row_pair_rx = torch.full((self.max_rows,), -1, dtype=torch.int32, device=dev)
        self.ids_rx = torch.empty(total, dtype=torch.int32, device=dev)
        self.pos_rx = torch.empty(total, dtype=torch.int32, device=dev)
        self.tiles = torch.empty(El + 1, dtype=torch.int32, device=dev)
        self.pos_dest = torch.empty(n, k, dtype=torch.int32, device=dev)
        self.dest_off = torch.empty(world + 1, dtype=torch.int32, device=dev)
        # the dispatch (possibly on the comm stream) and the receive-side regroup
        # (main stream) each own their permute scratch
        self.scratch = torch.zeros(ops.permute_scratch_ints(total, 1, El), dtype=torch.int32,
                                   device=dev)
        self.scratch_tx = torch.zeros(ops.permute_scratch_ints(n, k, world), dtype=torch.int32,
                                      device=dev)
        self.hsh = torch.empty(n, max(S, 1) * ep, dtype=bf, device=dev)
        # displaced: the dispatch in the windows and the new one coexist per layer
        per_layer = 2 if strategy is Strategy.DISPLACED else 1
        self.payloads = [[_EPPayload(n, k, dev) for _ in range(per_layer)] for _ in range(L)]
        # this rank's pair rows / gates / ids live in its window (the expert ranks
        # write them); with conditional communication they are the token cache's
        rows, gates, ids = self.win.pair_views(n)
        self.pair_rows, self.pair_gates, self.pair_ids = rows, gates, ids
        self.cache = TokenCache(L, n, k, cfg.hidden_dim, device=dev, rows=rows, gates=gates,
                                expert_ids=ids) \
            if policy.cond_strategy is not CondStrategy.OFF else None
        self.counters = torch.zeros(cfg.num_steps, L, 2, dtype=torch.int64, device=dev)
        self.status = torch.empty(4, dtype=torch.int32, device=dev)
        self.sync_layers = select_sync_layers(policy.sync_strategy, L, policy.explicit_layers)
        self.graph = None
        self._wait_events = []
        self._event_pool = []
        self._comm_events = []
        self._comm_pool = []
        self._join_events = []
        self._pool_next = 0
        self._expert_events = []
        self._expert_pool = []
        self.launches_per_run = 0

    # --------------------------------------------------------------- helpers
    def _slot(self, layer):
        return self.pair_rows[layer], self.pair_gates[layer]

    def _peers(self):
        return range(self.world)

    # ---------------------------------------------------------- comm stream
    def _send_overlapped(self, step, layer, p, decided):
        """The asynchronous stage's dispatch on the comm stream, ordered after
        the gate (main) by an event."""
        g = self.grp
        self._ev_id += 1
        fork = self._ev_id
        g.stream_op("record", "main", fork)
        g.stream_op("wait_event", "comm", fork)
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record()
            self.comm.wait_event(ev)
        g.stream = "comm"
        try:
            if self.cuda:
                with torch.cuda.stream(self.comm):
                    self._send(step, layer, p, force=False, decided=decided, timed=False)
                    done = torch.cuda.Event()
                    done.record()
            else:
                self._send(step, layer, p, force=False, decided=decided, timed=False)
                done = None
        finally:
            g.stream = "main"
        self._ev_id += 1
        g.stream_op("record", "comm", self._ev_id)
        self._comm_pending = (done, self._ev_id)

    def _join_comm(self):
        """Main waits for the outstanding comm-stream send (its rows are read
        from u16 / the payload, which the main stream is about to reuse)."""
        if self._comm_pending is None:
            return
        done, eid = self._comm_pending
        self._comm_pending = None
        self.grp.stream_op("wait_event", "main", eid)
        if not self.cuda:
            return
        evs = self._comm_begin()
        torch.cuda.current_stream().wait_event(done)
        if evs is not None:
            evs[1].record()
            self._join_events.append(evs)

    def _comm_begin(self):
        """Graph-safe event before an exchange kernel (dispatch send / regroup):
        on this single-stream rank they sit on the critical path, so their
        time counts as exposed all-to-all time next to the flag waits."""
        if not self.time_waits:
            return None
        i = self._pool_next
        self._pool_next += 1
        if i >= len(self._comm_pool):
            self._comm_pool.append((ops.DeviceEvent(), ops.DeviceEvent()))
        a, b = self._comm_pool[i]
        a.record()
        return a, b

    def _comm_end(self, evs):
        if evs is not None:
            evs[1].record()
            self._comm_events.append(evs)

    def _timed_wait(self, addrs, value):
        if self.time_waits:
            i = len(self._wait_events)
            if i >= len(self._event_pool):
                self._event_pool.append((ops.DeviceEvent(), ops.DeviceEvent()))
            a, b = self._event_pool[i]
            a.record()
        self.grp.wait(addrs, value)
        if self.time_waits:
            b.record()
            self._wait_events.append((a, b))

    def _reset_state(self, x0_device=None):
        cfg = self.cfg
        ops.status_reset(self.status)
        self.counters.zero_()
        x0 = x0_device
        if x0 is None:
            x0 = torch.as_tensor(self.x0.values).to(device=self.dev, dtype=torch.float32).contiguous()
        ops.pack_rows(x0, self.hp, self.x32, self.x16)
        if self.cache is not None:
            self.cache.has_subset.zero_()
        L = cfg.num_layers
        self.slot_gen = [None] * L
        self.deferred = [None] * L    # payload whose combine is assembled at next stage l
        self.disp = [None] * L        # displaced: (payload in the windows, processed at sync)
        self.pending = None
        self.occupied = set()
        self.peak_buffer_bytes = 0
        self.records, self.dispatch_log, self.combine_log = [], [], []
        self._wait_events = []
        self._comm_events = []
        self._join_events = []
        self._pool_next = 0
        self._expert_events = []
        self._comm_pending = None

    def _track(self, layer, kind="c"):
        self.occupied.add((kind, layer))
        slot_bytes = self.cfg.total_rows * self.cfg.hidden_dim * self.cluster.bytes_per_element
        self.peak_buffer_bytes = max(self.peak_buffer_bytes, len(self.occupied) * slot_bytes)

    def _stage_is_sync(self, step, layer):
        if self.strategy is Strategy.SYNCHRONOUS:
            return True
        if is_sync_step(step, self.policy.warmup, self.policy.period):
            return True
        if layer in self.sync_layers:
            return True
        if self.strategy is Strategy.DISPLACED:
            return self.disp[layer] is None or self.slot_gen[layer] is None
        return self.slot_gen[layer] is None

    def _payload(self, layer):
        pair = self.payloads[layer]
        if self.strategy is Strategy.DISPLACED and self.disp[layer] is not None:
            return pair[1] if self.disp[layer][0] is pair[0] else pair[0]
        return pair[0]

    # ------------------------------------------------------------- exchange
    def _send(self, step, layer, p: _EPPayload, force, decided=False, timed=True):
        """decide (unless the gate launch already took it) + dispatch all-to-all
        send of layer `layer`."""
        g, me, D = self.grp, self.rank, self.world
        if self.cache is not None:
            if not decided:
                self.cache.decide_into(layer, step, p.ids, self.policy, force, p.active, p.write,
                                       row0=self.r0)
            act = p.active
        else:
            act = None
        # my regions in every destination window must have been consumed
        wait = self._timed_wait if timed else g.wait
        wait([g.flag("rx_free", me, layer, d) for d in self._peers()], 1)
        g.write([g.flag("rx_free", me, layer, d) for d in self._peers()], 0)
        rx_rows = _u64_array([g.rx_rows(d, layer, me) for d in self._peers()])
        rx_meta = _u64_array([g.rx_meta(d, layer, me) for d in self._peers()])
        rx_cnt = _u64_array([g.rx_count(d, layer, me) for d in self._peers()])
        evs = self._comm_begin() if timed else None
        _lib.call("dice_ep_dispatch", p.ids.data_ptr(), p.gates.data_ptr(),
                  None if act is None else act.data_ptr(),
                  self.n, self.k, self.E, D, me, self.u16.data_ptr(), self.hp,
                  self.pos_dest.data_ptr(), self.dest_off.data_ptr(),
                  self.counters[step, layer].data_ptr(), self.r0, self.cfg.total_rows,
                  self.scratch_tx.data_ptr(), rx_rows, rx_meta, rx_cnt, ops._stream())
        self._comm_end(evs)
        g.data("write", [("rx", d, layer, me) for d in self._peers()])
        self._uread += 1
        g.data("uread", [], gen=self._uread)       # the send kernel read u16 / the payload
        g.write([g.flag("rx_ready", d, layer, me) for d in self._peers()], 1)
        p.layer, p.gen = layer, step
        self.dispatch_log.append((step, layer))

    def _expert(self, p: _EPPayload, shared_layer=None):
        """Expert side of dispatch(p.layer): wait for every source, grouped FFN,
        rows (with gates and expert ids) stored straight into their home ranks'
        pair rows by the GEMM2 epilogue. shared_layer: that layer's
        shared-expert GEMM1 (u16 -> hsh) rides in the expert GEMM1 launch."""
        g, me, layer = self.grp, self.rank, p.layer
        # as a home: every read of this layer's pair rows precedes this point in
        # the schedule (the rows are next written by this expert call), so free
        # them for every expert rank
        g.write([g.flag("cx_free", r, layer, me) for r in self._peers()], 1)
        self._timed_wait([g.flag("rx_ready", me, layer, s) for s in self._peers()], 1)
        g.write([g.flag("rx_ready", me, layer, s) for s in self._peers()], 0)
        # as an expert rank: every home has freed its rows of this layer
        self._timed_wait([g.flag("cx_free", me, layer, h) for h in self._peers()], 1)
        g.write([g.flag("cx_free", me, layer, h) for h in self._peers()], 0)
        lw = self.model.layers[layer]
        homes = self._peers()
        rows = _u64_array([g.cx_rows(h, layer) for h in homes])
        gates = _u64_array([g.cx_gates(h, layer) for h in homes])
        ids = _u64_array([g.cx_ids(h, layer) for h in homes])
        hn = (ctypes.c_int64 * len(self.shard_n))(*self.shard_n)
        evs = self._comm_begin()
        _lib.call("dice_ep_regroup", g.rx_rows(me, layer, 0), g.rx_meta(me, layer, 0),
                  g.rx_count(me, layer, 0), self.world, self.cap, self.El, self.hp,
                  self.ids_rx.data_ptr(), self.pos_rx.data_ptr(), self.tiles.data_ptr(),
                  self.scratch.data_ptr(), self.x_perm.data_ptr(), self.row_pair_rx.data_ptr(),
                  ops._stream())
        self._comm_end(evs)
        if self.time_experts:
            i = len(self._expert_events)
            if i >= len(self._expert_pool):
                self._expert_pool.append((ops.DeviceEvent(), ops.DeviceEvent()))
            e0, e1 = self._expert_pool[i]
            e0.record()
        _lib.call("dice_ep_expert_ffn", self.x_perm.data_ptr(), self.max_rows,
                  g.rx_meta(me, layer, 0), self.cap, self.world, self.El, self.hp, self.ep,
                  self.k, lw.w1_t.data_ptr(), lw.w2_t.data_ptr(), self.tiles.data_ptr(),
                  self.hbuf.data_ptr(), self.row_pair_rx.data_ptr(), rows, gates, ids, hn,
                  *self._shared_args(shared_layer), ops._stream())
        if self.time_experts:
            e1.record()
            self._expert_events.append((e0, e1, p.gen, layer, shared_layer is not None))
        g.data("read", [("rx", me, layer, s) for s in self._peers()])
        g.data("write", [("cx", h, layer, me) for h in self._peers()], gen=p.gen)
        g.write([g.flag("rx_free", s, layer, me) for s in self._peers()], 1)
        g.write([g.flag("cx_ready", h, layer, me) for h in self._peers()], 1)
        self.deferred[layer] = p
        self.slot_gen[layer] = p.gen          # the combine is in flight
        self.combine_log.append((p.gen, layer))

    def _discard(self, p: _EPPayload):
        """Expert side of a dispatch that is never processed (displaced, superseded
        by a sync stage or left at the end of the run): release the receive
        regions so the handshake state returns to its initial values."""
        g, me, layer = self.grp, self.rank, p.layer
        self._timed_wait([g.flag("rx_ready", me, layer, s) for s in self._peers()], 1)
        g.write([g.flag("rx_ready", me, layer, s) for s in self._peers()], 0)
        g.data("read", [("rx", me, layer, s) for s in self._peers()])
        g.write([g.flag("rx_free", s, layer, me) for s in self._peers()], 1)

    def _shared_args(self, shared_layer):
        if shared_layer is None:
            return (None, 0, None, 0, None)
        ws1 = self.model.layers[shared_layer].ws1_t
        return (self.u16.data_ptr(), self.n, ws1.data_ptr(), ws1.shape[0], self.hsh.data_ptr())

    def _assemble(self, layer):
        """Combine arrival at the home rank: every expert rank has stored its
        rows into this layer's pair rows (TokenCache.assemble needs no kernel:
        the rows are the cache, inactive pairs keep their cached entries)."""
        p = self.deferred[layer]
        if p is None:
            return
        g, me = self.grp, self.rank
        self._timed_wait([g.flag("cx_ready", me, layer, r) for r in self._peers()], 1)
        g.write([g.flag("cx_ready", me, layer, r) for r in self._peers()], 0)
        g.data("arrive", [("cx", me, layer, r) for r in self._peers()])
        self.deferred[layer] = None

    def _flush_pending(self):
        prev, self.pending = self.pending, None
        if prev is not None:
            self._expert(prev)
            self._track(prev.layer)

    def _consume(self, layer, step, gen, gemm1_done=False):
        """u + (shared + sum_s g_s row_s) over the layer's pair rows (step `gen`'s
        combine; the rows are freed at the layer's next expert call)."""
        lw = self.model.layers[layer]
        rows, gates = self._slot(layer)
        if self.S > 0:
            if not gemm1_done:
                ops.gemm(ops.EPI_GELU_BF16, self.u16, lw.ws1_t, out_bf16=self.hsh)
            ops.gemm_consume(self.hsh, lw.ws2_t, self.u32, rows, gates, self.h32, self.h16)
        else:
            ops.consume_rows(self.u32, rows, gates, self.h32, self.h16)
        self.grp.data("consume", [("cx", self.rank, layer, r) for r in self._peers()], gen=gen)
        self.records.append(StalenessRecord(layer=layer, used_step=step, generated_step=gen))

    def _run_step(self, step):
        cfg = self.cfg
        for layer in range(cfg.num_layers):
            lw = self.model.layers[layer]
            hin32, hin16 = (self.x32, self.x16) if layer == 0 else (self.h32, self.h16)
            self._join_comm()      # the previous stage's send read u16 / its payload
            self.grp.data("uwrite", [], gen=self._uread)   # local_block overwrites u16
            ops.gemm(ops.EPI_GELU_RESID, hin16, lw.w_mix_t, out_f32=self.u32,
                     out_bf16=self.u16, residual=hin32)
            sync = self._stage_is_sync(step, layer)
            if sync:
                self._flush_pending()
            self._assemble(layer)            # previous step's combine, before decide(layer)
            p = self._payload(layer)
            # the conditional-communication decision rides in the gate launch
            dec = None
            if self.cache is not None:
                dec = self.cache.decide_args(layer, step, self.policy, sync, p.active, p.write,
                                             row0=self.r0)
            ops.gate_topk(self.u32, lw.w_gate_t, self.k, p.ids, p.gates, None, self.status,
                          step, layer, decide=dec)
            decided = dec is not None
            if sync:
                old = self.disp[layer]
                if old is not None and not old[1]:
                    self._discard(old[0])    # superseded, never processed (schedules.py:336)
                self._send(step, layer, p, force=True, decided=decided)
                self._expert(p, shared_layer=layer if self.merge_gemm1 else None)
                self._assemble(layer)
                if self.strategy is Strategy.DISPLACED:
                    self.disp[layer] = (p, True)
                    self._track(layer, "d")
                    self._track(layer)
                elif self.strategy is Strategy.INTERWEAVED:
                    self._track(layer)
                self._consume(layer, step, step, gemm1_done=self.merge_gemm1)
            elif self.strategy is Strategy.DISPLACED:
                gen = self.slot_gen[layer]
                old, processed = self.disp[layer]
                # consume the pair rows (step s-2's combine) before the old
                # dispatch's combine overwrites them
                self._consume(layer, step, gen)
                if processed:
                    # the reference re-processes the sync stage's dispatch; its
                    # rows are already in the slot, its combine bytes count again
                    self.combine_log.append((old.gen, layer))
                else:
                    self._expert(old)
                self._track(layer)
                self._send(step, layer, p, force=False, decided=decided)
                self.disp[layer] = (p, False)
                self._track(layer, "d")
            else:
                gen = self.slot_gen[layer]
                if self.overlap_dispatch:
                    self._send_overlapped(step, layer, p, decided)
                else:
                    self._send(step, layer, p, force=False, decided=decided)
                prev, self.pending = self.pending, p
                merged = self.merge_gemm1 and prev is not None
                if prev is not None:
                    self._expert(prev, shared_layer=layer if merged else None)
                    self._track(prev.layer)
                self._consume(layer, step, gen, gemm1_done=merged)
        self._flush_pending()
        ops.denoise(self.x32, self.x16, self.h32, cfg.step_size, self.status, step)

    def _drain(self):
        """Assemble every outstanding combine so all flags return to their
        initial state (the run stays replayable)."""
        for layer in range(self.cfg.num_layers):
            self._assemble(layer)
            if self.disp[layer] is not None and not self.disp[layer][1]:
                self._discard(self.disp[layer][0])
                self.disp[layer] = None

    def device_bytes(self) -> int:
        """Physical device bytes of this rank's run: its buffers, payloads, token
        cache and its exchange window (not the model weights)."""
        seen, total = set(), int(self.win.nbytes)

        def visit(v, depth):
            nonlocal total
            if isinstance(v, torch.Tensor):
                if v.is_cuda and v.untyped_storage().data_ptr() not in seen:
                    seen.add(v.untyped_storage().data_ptr())
                    total += v.untyped_storage().nbytes()
            elif isinstance(v, (list, tuple)):
                for x in v:
                    visit(x, depth)
            elif depth < 2 and isinstance(v, (_EPPayload, TokenCache)):
                for x in vars(v).values():
                    visit(x, depth + 1)

        for key, v in vars(self).items():
            if key != "model":
                visit(v, 0)
        return total

    # ------------------------------------------------------------- run API
    def launch(self, x0_device=None):
        if self.graph is not None:
            if x0_device is not None and x0_device.data_ptr() != self._x0_graph.data_ptr():
                self._x0_graph.copy_(x0_device)
            self.graph.replay()
            return
        c0 = _lib.launch_count[0]
        self._reset_state(x0_device)
        for step in range(self.cfg.num_steps):
            self._run_step(step)
        self._join_comm()
        self._drain()
        self.launches_per_run = _lib.launch_count[0] - c0

    def sample(self, x0_host: torch.Tensor) -> torch.Tensor:
        """Serving entry for this rank's shard: x0 rows from (pinned) host memory
        -> final latent rows in host memory."""
        if not hasattr(self, "_final_host"):
            self._x0_stage = (self._x0_graph if self.graph is not None else
                              torch.empty(self.n, self.cfg.hidden_dim, dtype=torch.float32,
                                          device=self.dev))
            self._final_host = torch.empty(self.n, self.cfg.hidden_dim, dtype=torch.float32,
                                           pin_memory=True)
        self._x0_stage.copy_(x0_host, non_blocking=True)
        self.launch(self._x0_stage)
        self._final_host.copy_(self.x32[:, :self.cfg.hidden_dim], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self._final_host

    def capture(self):
        """Capture one whole sampling run into a CUDA graph. The schedule's
        control flow is host-deterministic and every buffer is static, so the
        graph replays the identical kernel sequence; x0 is read from a static
        staging buffer (see sample()). The warm-up run uses the capture stream
        so per-stream library state (tensor maps, kernel attributes) exists before capture."""
        self._x0_graph = torch.as_tensor(self.x0.values).to(
            device=self.dev, dtype=torch.float32).contiguous().clone()
        self._cap_stream = torch.cuda.Stream(device=self.dev)
        self._cap_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self._cap_stream):
            self.launch(self._x0_graph)          # warm: kernel attributes, tensor maps
        torch.cuda.synchronize()
        # no garbage collection inside the capture: freeing an earlier runner's
        # graph or events mid-capture would invalidate it
        import gc
        gc.collect()
        gc.disable()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self._cap_stream):
                self.launch(self._x0_graph)
        finally:
            gc.enable()
        torch.cuda.synchronize()
        self.graph = g
        return self

    def finish(self, reduce=True) -> RunResult:
        """Status + counters; bytes / pairs summed over ranks (torch.distributed)."""
        import torch.distributed as dist
        cfg = self.cfg
        status = self.status.cpu().tolist()
        cdev = "cuda" if self.world > 1 and dist.get_backend(self.pg) == "nccl" else "cpu"
        bad = torch.tensor([status[0]], dtype=torch.int64, device=cdev)
        cnt = self.counters.to(cdev).clone()
        if reduce and self.world > 1:
            dist.all_reduce(bad, op=dist.ReduceOp.MIN, group=self.pg)
            dist.all_reduce(cnt, group=self.pg)
        bad, cnt = bad.cpu(), cnt.cpu()
        if int(bad.item()) != INT32_MAX:
            raise NumericalDivergenceError(f"non-finite values at step {int(bad.item())}",
                                           step=int(bad.item()))
        cnt = cnt.numpy()
        row_bytes = cfg.hidden_dim * self.cluster.bytes_per_element
        dispatch_bytes = int(sum(cnt[s, l, 1] for s, l in self.dispatch_log)) * row_bytes
        combine_bytes = int(sum(cnt[s, l, 1] for s, l in self.combine_log)) * row_bytes
        per_step_active = [int(v) for v in cnt[:, :, 0].sum(axis=1)]
        per_step_total = [cfg.num_layers * cfg.total_rows * self.k] * cfg.num_steps
        timeline = None
        if self._wait_events:
            waits = sum(a.elapsed_ms(b) for a, b in self._wait_events) * 1e-3
            kernels = sum(a.elapsed_ms(b) for a, b in self._comm_events) * 1e-3
            joins = sum(a.elapsed_ms(b) for a, b in self._join_events) * 1e-3
            # on the main stream: the flag waits, the exchange kernels issued on
            # it (blocking stages' dispatch, every receive-side regroup) and the
            # waits for the overlapped sends of the comm stream
            timeline = {"exposed_comm_seconds": waits + kernels + joins,
                        "comm_wait_seconds": waits, "comm_kernel_seconds": kernels,
                        "comm_join_seconds": joins}
        return RunResult(
            final=ActivationBlock(values=self.x32[:, :cfg.hidden_dim].clone(),
                                  generated_step=cfg.num_steps),
            timeline=timeline, staleness_records=self.records, strategy=self.strategy,
            policy=self.policy, seed=self.seed, model_hash=model_hash(self.model),
            x0_hash=hashlib.sha256(np.ascontiguousarray(
                torch.as_tensor(self.x0.values).cpu().numpy()).tobytes()).hexdigest(),
            config=cfg, cluster=self.cluster, dispatch_bytes=dispatch_bytes,
            combine_bytes=combine_bytes, peak_buffer_bytes=self.peak_buffer_bytes,
            active_pairs=sum(per_step_active), total_pairs=sum(per_step_total),
            per_step_active_pairs=per_step_active, per_step_total_pairs=per_step_total)

    def run(self) -> RunResult:
        self.launch()
        return self.finish()

    def close(self):
        torch.cuda.synchronize()
        self.graph = None
        self.grp.close()
        self.win.free()
