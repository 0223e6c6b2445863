"""Execution schedules on the GPU — drop-in for dicesim.schedules
(/root/reference/pkg/src/dicesim/schedules.py).

``run_sampling`` keeps the reference signature and RunResult fields. The
per-layer stage logic (synchronous / displaced / interweaved, selective and
periodic sync, conditional communication; schedules.py:319-457) is host
control flow; every value is produced by the sm_100a library, stream-ordered,
with no host synchronisation inside the run. Device-side counters and the
non-finite status word are read once at the end of the run.

Buffers (all HBM-resident, allocated once per runner):
* a dispatch payload = gate ids/gates, cond masks, permute positions/tile
  offsets, the row -> pair map and the expert-sorted bf16 token rows
  (DispatchPayload, 48-57);
* per layer, the pair rows bf16 [k, n, hp] and pair gates f32 [n, k]: the
  latest computed expert row and gate of every (token, slot) pair — the token
  cache's rows / gates when conditional communication is on (TokenCache,
  policies.py:142-208) — which together are the layer's combine slot
  (CombinePayload + LayerBuffers, 60-79). The expert GEMM2 epilogue writes
  them; the shared-FFN GEMM2 epilogue consumes them, u + (shared + sum g row).
"""
from __future__ import annotations

import dataclasses
import hashlib
from collections import Counter
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import ops
from .cluster import ClusterConfig, build_placement
from .errors import ContractError, NumericalDivergenceError
from .model import ActivationBlock, RouteDecision, ToyModel, model_hash, similarity_from_sums
from .policies import (CondStrategy, PolicyConfig, TokenCache, is_sync_step,
                       select_sync_layers)

INT32_MAX = 2 ** 31 - 1


class Strategy(Enum):
    SYNCHRONOUS = "synchronous"
    DISPLACED = "displaced"
    INTERWEAVED = "interweaved"


@dataclass(frozen=True)
class StalenessRecord:
    layer: int
    used_step: int
    generated_step: int

    @property
    def staleness(self) -> int:
        return self.used_step - self.generated_step


@dataclass
class RunResult:
    """Same fields as schedules.py:92-129. ``timeline`` holds measured CUDA-event
    stage timings when the run was timed (else None)."""
    final: ActivationBlock
    timeline: object
    staleness_records: list
    strategy: Strategy
    policy: PolicyConfig
    seed: int
    model_hash: str
    x0_hash: str
    config: object
    cluster: ClusterConfig
    dispatch_bytes: int
    combine_bytes: int
    peak_buffer_bytes: int
    active_pairs: int
    total_pairs: int
    per_step_active_pairs: list
    per_step_total_pairs: list
    step_inputs: list | None = None
    step_routes: list | None = None
    gpu_seconds: float | None = None
    similarity: object = None     # StepSimilarity of the run (track_similarity)

    @property
    def total_comm_bytes(self) -> int:
        return self.dispatch_bytes + self.combine_bytes

    @property
    def makespan_seconds(self) -> float | None:
        return self.gpu_seconds

    @property
    def comm_stall_seconds(self) -> float:
        return 0.0 if self.timeline is None else self.timeline.get("exposed_comm_seconds", 0.0)

    def staleness_histogram(self) -> dict:
        counts = Counter(rec.staleness for rec in self.staleness_records)
        return dict(sorted(counts.items()))


class GpuTimeline:
    """Measured stage timeline in the reference's export schema
    (cluster.py:132-138, 210-216): events {device, kind, start, end, label},
    seconds from the start of the run, from CUDA events on the stream."""

    def __init__(self, events, device=0):
        self.events = events
        self.device = device

    def export(self) -> list:
        return [dict(device=self.device, kind=k, start=a, end=b, label=l) for k, a, b, l in self.events]

    def to_json(self) -> str:
        import json
        return json.dumps({"schema_version": 1, "events": self.export()}, separators=(",", ":"))

    def makespan(self) -> float:
        return max((b for _, _, b, _ in self.events), default=0.0)

    def get(self, key, default=None):
        return {"makespan_seconds": self.makespan()}.get(key, default)


class _Payload:
    """Device buffers of one dispatch (DispatchPayload, schedules.py:48-57).
    max_rows: rows of the expert-sorted buffer (tile-contiguous experts, or E
    capacity regions of the fused router)."""

    def __init__(self, n, k, E, hp, max_rows, device):
        self.ids = torch.zeros(n, k, dtype=torch.int32, device=device)
        self.gates = torch.zeros(n, k, dtype=torch.float32, device=device)
        self.active = torch.ones(n, k, dtype=torch.uint8, device=device)
        self.write = torch.zeros(n, k, dtype=torch.uint8, device=device)
        self.pos = torch.zeros(n, k, dtype=torch.int32, device=device)
        self.tiles = torch.zeros(E + 1, dtype=torch.int32, device=device)
        self.x_perm = torch.empty(max_rows, hp, dtype=torch.bfloat16, device=device)
        # permuted row -> (token, slot) pair (-1 on padding rows), for the expert
        # GEMM2's pair-row stores
        self.row_pair = torch.full((max_rows,), -1, dtype=torch.int32, device=device)
        self.layer = -1
        self.gen = -1
        self.done = None     # side-stream event: expert FFN of this payload finished


class DeviceRunner:
    """One sampling run on one GPU: owns buffers, cache, counters (ScheduleRunner,
    schedules.py:142-490)."""

    def __init__(self, model: ToyModel, x0: ActivationBlock, strategy: Strategy,
                 policy: PolicyConfig, cluster: ClusterConfig, seed: int, *,
                 record_inputs: bool = False, record_routes: bool = False,
                 time_experts: bool = False, overlap: bool = False, timeline: bool = False,
                 time_ops: bool = False, record_filter=None, record_outputs: bool = False,
                 track_similarity: bool = False):
        """track_similarity: accumulate step_similarity's sums on the device
        during the run (each layer's previous-step MoE input and top-1 ids kept
        in HBM, one fused compare-and-roll launch pair per stage; no host
        copies) -> ``RunResult.similarity``.
        record_inputs / record_routes: per (step, layer) MoE inputs u and
        routes (+ the conditional-communication masks in ``step_masks``), as
        run_sampling(record_*=True); ``record_filter(step, layer)`` limits the
        recorded inputs (others are None), ``record_outputs`` also records the
        layer outputs h at those stages (``step_outputs``)."""
        cfg = model.config
        if not isinstance(strategy, Strategy):
            raise ContractError(f"strategy must be a Strategy, got {strategy!r}")
        if x0.generated_step != 0:
            raise ContractError(f"x0 must carry generated_step 0, got {x0.generated_step}")
        expected = (cfg.total_rows, cfg.hidden_dim)
        if tuple(x0.values.shape) != expected:
            raise ContractError(f"x0 shape {tuple(x0.values.shape)} does not match model {expected}")
        if model.num_local_experts != cfg.num_experts:
            raise ContractError("single-device runner needs every routed expert resident")
        if policy.cond_strategy is CondStrategy.RANDOM and policy.cond_seed is None:
            policy = dataclasses.replace(policy, cond_seed=seed)   # schedules.py:158-159
        build_placement(cfg.num_experts, cluster.num_devices, cfg.total_rows)  # validates E % D
        self.model, self.cfg, self.x0 = model, cfg, x0
        self.strategy, self.policy, self.cluster, self.seed = strategy, policy, cluster, seed
        self.record_inputs, self.record_routes = record_inputs, record_routes
        self.record_filter = record_filter or (lambda step, layer: True)
        self.record_outputs = record_outputs
        self.time_experts = time_experts
        # time_ops: graph-safe CUDA events around every library op of the run
        # (per-op device time inside the real step; costs a few % of the step)
        self.time_ops = time_ops
        self._op_events, self._op_pool = [], []
        self.want_timeline = timeline
        dev = model.device
        self.dev = dev
        n, k, E, S = cfg.total_rows, cfg.top_k, cfg.num_experts, cfg.num_shared
        hp, ep = model.hp, model.ep
        self.n, self.k, self.E, self.S, self.hp, self.ep = n, k, E, S, hp, ep
        self.max_rows = ops.permute_max_rows(n, k, E)
        # E = 8 / 16: the gate launch also permutes (dice_gate_route); expert
        # e's rows live in a capacity region of cap rows (>= n: a token routes
        # to an expert at most once)
        self.fused_route = E in (8, 16) and k <= E
        self.cap = (n + 255) // 256 * 256
        perm_rows = max(E * self.cap, self.max_rows) if self.fused_route else self.max_rows
        f32, bf = torch.float32, torch.bfloat16
        self.x32 = torch.zeros(n, hp, dtype=f32, device=dev)
        self.x16 = torch.zeros(n, hp, dtype=bf, device=dev)
        self.h32 = torch.zeros(n, hp, dtype=f32, device=dev)
        self.h16 = torch.zeros(n, hp, dtype=bf, device=dev)
        self.u32 = torch.zeros(n, hp, dtype=f32, device=dev)
        self.u16 = torch.zeros(n, hp, dtype=bf, device=dev)
        self.hbuf = torch.empty(self.max_rows, ep, dtype=bf, device=dev)
        self.hsh = torch.empty(n, max(S, 1) * ep, dtype=bf, device=dev)
        self.scores = torch.empty(n, E, dtype=f32, device=dev) if record_routes else None
        L = cfg.num_layers
        if strategy is Strategy.SYNCHRONOUS:
            self.payloads = [_Payload(n, k, E, hp, perm_rows, dev)]
        elif strategy is Strategy.INTERWEAVED:
            self.payloads = [_Payload(n, k, E, hp, perm_rows, dev) for _ in range(3)]
        else:
            self.payloads = [[_Payload(n, k, E, hp, perm_rows, dev) for _ in range(2)]
                             for _ in range(L)]
        self.cache = None
        if policy.cond_strategy is not CondStrategy.OFF:
            self.cache = TokenCache(L, n, k, cfg.hidden_dim, device=dev)
            self.pair_rows, self.pair_gates = self.cache.rows, self.cache.gates
            self.pair_ids = self.cache.expert_ids
        else:
            nslots = 1 if strategy is Strategy.SYNCHRONOUS else L
            self.pair_rows = torch.zeros(nslots, k, n, hp, dtype=bf, device=dev)
            self.pair_gates = torch.zeros(nslots, n, k, dtype=f32, device=dev)
            self.pair_ids = None
        self.scratch = torch.zeros(ops.permute_scratch_ints(n, k, E), dtype=torch.int32, device=dev)
        self.track_similarity = track_similarity
        if track_similarity:
            self.sim_prev = torch.zeros(L, n, hp, dtype=f32, device=dev)
            self.sim_top = torch.zeros(L, n, dtype=torch.int32, device=dev)
            self.sim_sums = torch.zeros(L, max(cfg.num_steps - 1, 1), 4, dtype=torch.float64,
                                        device=dev)
            self.sim_sink = torch.zeros(4, dtype=torch.float64, device=dev)
            self.sim_part = torch.empty(ops.similarity_partial_words(), dtype=torch.float64,
                                        device=dev)
        self.route_state = (torch.zeros(ops.route_state_words(n), dtype=torch.int64, device=dev)
                            if self.fused_route else None)
        self.counters = torch.zeros(cfg.num_steps, L, 2, dtype=torch.int64, device=dev)
        self.status = torch.empty(4, dtype=torch.int32, device=dev)
        self.sync_layers = select_sync_layers(policy.sync_strategy, L, policy.explicit_layers)
        self._expert_events = []
        self._event_pool = []
        self.graph = None
        self.launches_per_run = 0
        # interweaved: the pending dispatch's expert FFN + cache merge run on a side
        # stream, concurrently with the next stage's shared FFN / consume on the
        # main stream (the intra-GPU analogue of the interweaved overlap window)
        self._marks, self._mark_pool = [], []
        self.side = None
        if overlap and strategy is Strategy.INTERWEAVED and str(dev).startswith("cuda") and not timeline:
            self.side = torch.cuda.Stream(device=dev)
        # the processed dispatch's expert GEMM1 and the stage's shared-expert GEMM1
        # are independent: one persistent launch for both
        self.merge_gemm1 = (S > 0 and self.side is None
                            and strategy in (Strategy.SYNCHRONOUS, Strategy.INTERWEAVED))

    # ------------------------------------------------------------ helpers
    def _reset_state(self, x0_device=None):
        cfg = self.cfg
        ops.status_reset(self.status)
        self.counters.zero_()
        x0 = x0_device
        if x0 is None:
            x0 = torch.as_tensor(self.x0.values).to(device=self.dev, dtype=torch.float32).contiguous()
        ops.pack_rows(x0, self.hp, self.x32, self.x16)
        if self.cache is not None:
            # an unprimed token is due (policies.py:171), and every cache entry is
            # written at that refresh before it is read, so clearing the primed
            # flags resets the cache
            self.cache.has_subset.zero_()
        L = cfg.num_layers
        self.slot_gen = [None] * L          # generating step of each combine slot
        self.dispatch_slot = [None] * L     # displaced only
        self.pending = None                 # interweaved only
        self.slot_event = [None] * L        # side-stream event guarding slot[l] / cache[l]
        self.side_tail = None
        for p in (self.payloads if self.strategy is Strategy.INTERWEAVED else []):
            p.done = None
        self.occupied = set()
        self.peak_buffer_bytes = 0
        self.ring = 0
        self.records = []
        self.dispatch_log = []
        self.combine_log = []
        self.step_inputs, self.step_routes, self.step_masks, self.step_outputs = [], [], [], []
        self._expert_events = []  # (start, end, generated step, layer) of each expert-FFN launch
        self._marks = []
        self._op_events = []      # (op, start, end, step, layer) when time_ops

    def _mark(self, label):
        """Stage boundary for the measured timeline (graph-safe CUDA event)."""
        if not self.want_timeline:
            return
        i = len(self._marks)
        if i >= len(self._mark_pool):
            self._mark_pool.append(ops.DeviceEvent())
        ev = self._mark_pool[i]
        ev.record()
        self._marks.append((label, ev))

    def _op(self, name, step, layer):
        """Context bracketing one library op with graph-safe events (time_ops)."""
        runner = self

        class _Ctx:
            def __enter__(self_):
                if not runner.time_ops:
                    return
                i = len(runner._op_events)
                if i >= len(runner._op_pool):
                    runner._op_pool.append((ops.DeviceEvent(), ops.DeviceEvent()))
                self_.ev = runner._op_pool[i]
                self_.ev[0].record()

            def __exit__(self_, *a):
                if runner.time_ops:
                    self_.ev[1].record()
                    runner._op_events.append((name, self_.ev[0], self_.ev[1], step, layer))
        return _Ctx()

    def device_bytes(self) -> int:
        """Physical device bytes of the run's own buffers (activations, payloads,
        combine slots, token cache, scratch; not the model weights): every CUDA
        tensor reachable from the runner, its payloads and its cache, counted
        once per storage."""
        seen, total = set(), 0

        def visit(v, depth):
            nonlocal total
            if isinstance(v, torch.Tensor):
                if v.is_cuda and v.untyped_storage().data_ptr() not in seen:
                    seen.add(v.untyped_storage().data_ptr())
                    total += v.untyped_storage().nbytes()
            elif isinstance(v, (list, tuple)):
                for x in v:
                    visit(x, depth)
            elif depth < 2 and isinstance(v, (_Payload, TokenCache)):
                for x in vars(v).values():
                    visit(x, depth + 1)

        for key, v in vars(self).items():
            if key != "model":
                visit(v, 0)
        return total

    def op_times(self):
        """[(op, ms, step, layer)] of the last run / replay (time_ops)."""
        return [(n, a.elapsed_ms(b), s, l) for n, a, b, s, l in self._op_events]

    def _track(self, kind, layer):
        self.occupied.add((kind, layer))
        slot_bytes = self.cfg.total_rows * self.cfg.hidden_dim * self.cluster.bytes_per_element
        self.peak_buffer_bytes = max(self.peak_buffer_bytes, len(self.occupied) * slot_bytes)

    def _stage_is_sync(self, step, layer) -> bool:
        """schedules.py:406-416."""
        if self.strategy is Strategy.SYNCHRONOUS:
            return True
        if is_sync_step(step, self.policy.warmup, self.policy.period):
            return True
        if layer in self.sync_layers:
            return True
        if self.strategy is Strategy.DISPLACED:
            return self.dispatch_slot[layer] is None or self.slot_gen[layer] is None
        return self.slot_gen[layer] is None

    def _next_payload(self, layer):
        if self.strategy is Strategy.SYNCHRONOUS:
            return self.payloads[0]
        if self.strategy is Strategy.INTERWEAVED:
            p = self.payloads[self.ring]
            self.ring = (self.ring + 1) % len(self.payloads)
            if p.done is not None:       # the side stream may still read this buffer
                torch.cuda.current_stream().wait_event(p.done)
                p.done = None
            return p
        pair = self.payloads[layer]
        return pair[1] if self.dispatch_slot[layer] is pair[0] else pair[0]

    def _slot(self, layer):
        """(pair rows [k, n, hp], pair gates [n, k], cached ids or None) of a layer."""
        i = 0 if self.pair_rows.shape[0] == 1 else layer
        return (self.pair_rows[i], self.pair_gates[i],
                None if self.pair_ids is None else self.pair_ids[i])

    # -------------------------------------------------------------- stages
    def _dispatch(self, step, layer, p: _Payload, force: bool, decided: bool = False):
        """decide (policies.py:159-186) + permute/pack of the token rows that travel."""
        if self.cache is not None:
            if not decided:
                self.cache.decide_into(layer, step, p.ids, self.policy, force, p.active, p.write)
            act = p.active
        else:
            act = None
        if not self.fused_route:           # (else the gate launch permuted)
            with self._op("permute", step, layer):
                ops.route_permute(p.ids, act, self.u16, p.x_perm, p.pos, p.tiles,
                                  self.counters[step, layer], self.scratch, self.E,
                                  devices=self.cluster.num_devices, row0=0, rows_total=self.n,
                                  row_pair=p.row_pair)
        p.layer, p.gen = layer, step
        self.dispatch_log.append((step, layer))

    def _process(self, p: _Payload, side: bool = False, shared_layer=None):
        """Expert FFN on a dispatched payload + stale-cache merge into its
        combine slot (_process_dispatch, schedules.py:388-397). With side=True
        the work is enqueued on the side stream after the payload's dispatch."""
        if side and self.side is not None:
            ready = torch.cuda.Event()
            ready.record()
            self.side.wait_event(ready)
            with torch.cuda.stream(self.side):
                self._process_body(p, shared_layer)
                done = torch.cuda.Event()
                done.record()
            p.done = done
            self.slot_event[p.layer] = done
            self.side_tail = done
            return
        self._join_side()
        self._process_body(p, shared_layer)

    def _join_side(self):
        """Main stream waits for all side-stream work (shared expert scratch)."""
        if self.side_tail is not None:
            torch.cuda.current_stream().wait_event(self.side_tail)
            self.side_tail = None

    def _process_body(self, p: _Payload, shared_layer=None):
        """Expert FFN of a dispatch; the GEMM2 epilogue stores every computed
        pair's row / gate / id into the layer's pair rows (the stale-cache merge
        of TokenCache.assemble, policies.py:188-208, needs no kernel: inactive
        pairs keep their cached entries). shared_layer: also run that layer's
        shared-expert GEMM1 (u16 -> hsh) inside the expert GEMM1 launch."""
        self._mark(f"expert s{p.gen} L{p.layer}")
        lw = self.model.layers[p.layer]
        if self.time_experts:
            i = len(self._expert_events)
            if i >= len(self._event_pool):
                self._event_pool.append((ops.DeviceEvent(), ops.DeviceEvent()))
            e0, e1 = self._event_pool[i]
            e0.record()
        name = "grouped_ffn" if shared_layer is None else "grouped_ffn+shared_gemm1"
        rows, gates, ids = self._slot(p.layer)
        stride = self.cap if self.fused_route else 0
        with self._op(name, p.gen, p.layer):
            if shared_layer is None:
                ops.expert_gemm1_with_shared(p.x_perm, lw.w1_t, self.E, p.tiles, self.hbuf,
                                             self.u16[:0], lw.w1_t, self.hsh, group_stride=stride)
            else:
                ops.expert_gemm1_with_shared(p.x_perm, lw.w1_t, self.E, p.tiles, self.hbuf,
                                             self.u16, self.model.layers[shared_layer].ws1_t,
                                             self.hsh, group_stride=stride)
            ops.expert_gemm2_pairs(self.hbuf, lw.w2_t, self.E, p.tiles, p.row_pair, p.gates,
                                   p.ids, rows, gates, ids, pair_group_stride=stride)
        if self.time_experts:
            e1.record()
            self._expert_events.append((e0, e1, p.gen, p.layer, shared_layer is not None))
        self.slot_gen[p.layer] = p.gen
        self.combine_log.append((p.gen, p.layer))

    def _flush_pending(self, side=False):
        prev, self.pending = self.pending, None
        if prev is not None:
            self._process(prev, side=side)
            self._track("c", prev.layer)

    def _consume(self, layer, step, gen, gemm1_done=False):
        """u + (shared + sum_s g_s row_s) fused into the shared-FFN GEMM2 epilogue
        over the layer's pair rows (_consume, schedules.py:308-317;
        combine_outputs, model.py:279-298)."""
        lw = self.model.layers[layer]
        rows, gates, _ = self._slot(layer)
        self._mark(f"shared+consume s{step} L{layer}")
        if self.S > 0:
            if not gemm1_done:
                with self._op("shared_gemm1", step, layer):
                    ops.gemm(ops.EPI_GELU_BF16, self.u16, lw.ws1_t, out_bf16=self.hsh)
            with self._op("shared_gemm2_consume", step, layer):
                ops.gemm_consume(self.hsh, lw.ws2_t, self.u32, rows, gates, self.h32, self.h16)
        else:
            ops.consume_rows(self.u32, rows, gates, self.h32, self.h16)
        self.records.append(StalenessRecord(layer=layer, used_step=step, generated_step=gen))

    def _run_step(self, step):
        cfg = self.cfg
        inputs_here, routes_here, masks_here, outputs_here = [], [], [], []
        for layer in range(cfg.num_layers):
            lw = self.model.layers[layer]
            hin32, hin16 = (self.x32, self.x16) if layer == 0 else (self.h32, self.h16)
            self._mark(f"local s{step} L{layer}")
            with self._op("local_gemm", step, layer):
                ops.gemm(ops.EPI_GELU_RESID, hin16, lw.w_mix_t, out_f32=self.u32,
                         out_bf16=self.u16, residual=hin32)
            self._mark(f"gate+dispatch s{step} L{layer}")
            sync = self._stage_is_sync(step, layer)
            if sync and self.strategy is Strategy.INTERWEAVED:
                self._flush_pending()
            if self.slot_event[layer] is not None:
                # slot[layer] / cache[layer] are written on the side stream
                torch.cuda.current_stream().wait_event(self.slot_event[layer])
                self.slot_event[layer] = None
            p = self._next_payload(layer)
            dec = None
            if self.cache is not None:
                dec = self.cache.decide_args(layer, step, self.policy, sync, p.active, p.write)
            with self._op("gate_route" if self.fused_route else "gate_decide", step, layer):
                if self.fused_route:
                    ops.gate_route(self.u32, lw.w_gate_t, self.k, p.ids, p.gates, p.x_perm,
                                   self.cap, p.pos, p.row_pair, p.tiles, self.counters[step, layer],
                                   self.route_state, self.scores, self.status, step, layer,
                                   decide=dec, devices=self.cluster.num_devices,
                                   rows_total=self.n)
                else:
                    ops.gate_topk(self.u32, lw.w_gate_t, self.k, p.ids, p.gates, self.scores,
                                  self.status, step, layer, decide=dec)
            decided = dec is not None
            if self.track_similarity:
                with self._op("step_similarity", step, layer):
                    ops.step_similarity(self.sim_prev[layer], self.u32, cfg.hidden_dim,
                                        self.sim_top[layer], p.ids,
                                        self.sim_sums[layer, step - 1] if step > 0
                                        else self.sim_sink, self.sim_part, roll=True)
            keep = self.record_filter(step, layer)
            if self.record_inputs:
                inputs_here.append(self.u32[:, :cfg.hidden_dim].cpu() if keep else None)
            if self.record_routes:
                routes_here.append(RouteDecision(p.ids.long().cpu(), p.gates.cpu(),
                                                 self.scores.cpu()))
                masks_here.append((p.active.bool().cpu(), p.write.bool().cpu())
                                  if self.cache is not None else None)
            if sync:
                self._dispatch(step, layer, p, force=True, decided=decided)
                self._process(p, shared_layer=layer if self.merge_gemm1 else None)
                if self.strategy is Strategy.DISPLACED:
                    self.dispatch_slot[layer] = p
                    self._track("d", layer)
                    self._track("c", layer)
                elif self.strategy is Strategy.INTERWEAVED:
                    self._track("c", layer)
                self._consume(layer, step, step, gemm1_done=self.merge_gemm1)
            elif self.strategy is Strategy.DISPLACED:
                self._dispatch(step, layer, p, force=False, decided=decided)
                old = self.dispatch_slot[layer]
                self.dispatch_slot[layer] = p
                self._track("d", layer)
                gen = self.slot_gen[layer]
                # consume the slot before the old dispatch overwrites it; cache
                # ops keep the reference order decide(new) -> assemble(old)
                self._consume(layer, step, gen)
                self._process(old)
                self._track("c", layer)
            else:
                self._dispatch(step, layer, p, force=False, decided=decided)
                prev, self.pending = self.pending, p
                merged = self.merge_gemm1 and prev is not None
                if prev is not None:
                    self._process(prev, side=True, shared_layer=layer if merged else None)
                    self._track("c", prev.layer)
                self._consume(layer, step, self.slot_gen[layer], gemm1_done=merged)
            if self.record_outputs:
                outputs_here.append(self.h32[:, :cfg.hidden_dim].cpu() if keep else None)
        if (self.strategy is Strategy.INTERWEAVED and self.pending is not None
                and step + 1 < cfg.num_steps):
            # the reference flushes the last layer's dispatch at the end of the
            # step (schedules.py:443); the combine slot is claimed here, and the
            # expert FFN itself runs at the next step's first asynchronous stage,
            # inside that stage's shared-GEMM1 launch (or before a synchronous
            # stage): the same values, since the FFN depends on the dispatched
            # rows only and layer L-1 is consumed no earlier than step s+1
            self._track("c", self.pending.layer)
        else:
            self._flush_pending(side=self.strategy is Strategy.INTERWEAVED)
        self._mark(f"denoise s{step}")
        with self._op("denoise", step, -1):
            ops.denoise(self.x32, self.x16, self.h32, cfg.step_size, self.status, step)
        self._mark(f"end s{step}")
        if self.record_inputs:
            self.step_inputs.append(inputs_here)
        if self.record_routes:
            self.step_routes.append(routes_here)
            self.step_masks.append(masks_here)
        if self.record_outputs:
            self.step_outputs.append(outputs_here)

    def launch(self, x0_device=None):
        """Enqueue the whole run (no host sync). ``x0_device`` (f32 [R, h] on
        the device) replaces the constructor's x0 for repeated sampling. With a
        captured graph this is one graph launch."""
        if self.graph is not None:
            if x0_device is not None and x0_device.data_ptr() != self._x0_graph.data_ptr():
                self._x0_graph.copy_(x0_device)
            self.graph.replay()
            return
        from . import _lib
        c0 = _lib.launch_count[0]
        self._reset_state(x0_device)
        for step in range(self.cfg.num_steps):
            self._run_step(step)
        self._join_side()
        self.launches_per_run = _lib.launch_count[0] - c0

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

    def sample(self, x0_host: torch.Tensor) -> torch.Tensor:
        """Serving entry: x0 from (pinned) host memory -> final latent in host
        memory. H2D, the full schedule and the D2H read are stream-ordered."""
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

    def sample_many(self, x0_hosts, out_hosts) -> None:
        """Serve a sequence of batches (x0_hosts[i] -> out_hosts[i], pinned host
        tensors [R, h] f32) with the copies off the critical path: batch i's H2D
        and batch i-1's D2H run on a copy stream while batch i-1 / i replay, via
        double-buffered device staging. Needs capture(). Returns when every
        output has landed in host memory."""
        if self.graph is None:
            raise ContractError("sample_many needs a captured run (capture())")
        h = self.cfg.hidden_dim
        if not hasattr(self, "_pipe"):
            mk = lambda: torch.empty(self.n, h, dtype=torch.float32, device=self.dev)
            ev = lambda: torch.cuda.Event()
            self._pipe = dict(copy=torch.cuda.Stream(device=self.dev),
                              inb=[mk(), mk()], outb=[mk(), mk()],
                              in_ready=[ev(), ev()], in_free=[ev(), ev()],
                              out_ready=[ev(), ev()], out_free=[ev(), ev()], used=[False] * 4)
        P = self._pipe
        main, copy = torch.cuda.current_stream(), P["copy"]
        for i, (xh, oh) in enumerate(zip(x0_hosts, out_hosts)):
            b = i & 1
            if P["used"][b]:
                copy.wait_event(P["in_free"][b])        # replay i-2 took its input
            with torch.cuda.stream(copy):
                P["inb"][b].copy_(xh, non_blocking=True)
                P["in_ready"][b].record(copy)
            main.wait_event(P["in_ready"][b])
            self._x0_graph.copy_(P["inb"][b])
            P["in_free"][b].record(main)
            P["used"][b] = True
            self.graph.replay()
            if P["used"][2 + b]:
                main.wait_event(P["out_free"][b])       # D2H of batch i-2 done
            P["outb"][b].copy_(self.x32[:, :h])
            P["out_ready"][b].record(main)
            P["used"][2 + b] = True
            copy.wait_event(P["out_ready"][b])
            with torch.cuda.stream(copy):
                oh.copy_(P["outb"][b], non_blocking=True)
                P["out_free"][b].record(copy)
        copy.synchronize()
        main.synchronize()

    def finish(self, gpu_seconds=None) -> RunResult:
        """One device->host read of status + counters; build the RunResult."""
        cfg = self.cfg
        status = self.status.cpu().tolist()
        if status[0] != INT32_MAX:
            raise NumericalDivergenceError(
                f"non-finite values at step {status[0]} (layer {status[1]})", step=status[0])
        cnt = self.counters.cpu().numpy()
        row_bytes = cfg.hidden_dim * self.cluster.bytes_per_element
        dispatch_bytes = int(sum(cnt[s, l, 1] for s, l in self.dispatch_log)) * row_bytes
        combine_bytes = int(sum(cnt[s, l, 1] for s, l in self.combine_log)) * row_bytes
        per_step_active = [int(v) for v in cnt[:, :, 0].sum(axis=1)]
        per_step_total = [cfg.num_layers * self.n * self.k] * cfg.num_steps
        final = ActivationBlock(values=self.x32[:, :cfg.hidden_dim].clone(),
                                generated_step=cfg.num_steps)
        timeline = None
        if self._marks:
            t0 = self._marks[0][1]
            times = [t0.elapsed_ms(ev) * 1e-3 for _, ev in self._marks]
            events = [("compute", times[i], times[i + 1], self._marks[i][0])
                      for i in range(len(self._marks) - 1)
                      if not self._marks[i][0].startswith("end ")]
            timeline = GpuTimeline(events, device=torch.cuda.current_device())
            gpu_seconds = timeline.makespan() if gpu_seconds is None else gpu_seconds
        elif self._expert_events:
            timeline = {"expert_ffn_ms": [ev[0].elapsed_ms(ev[1]) for ev in self._expert_events]}
        return RunResult(
            final=final, timeline=timeline, staleness_records=self.records,
            strategy=self.strategy, policy=self.policy, seed=self.seed,
            model_hash=model_hash(self.model),
            x0_hash=hashlib.sha256(
                np.ascontiguousarray(torch.as_tensor(self.x0.values).detach().cpu().numpy()
                                     ).tobytes()).hexdigest(),
            config=cfg, cluster=self.cluster, dispatch_bytes=dispatch_bytes,
            combine_bytes=combine_bytes, peak_buffer_bytes=self.peak_buffer_bytes,
            active_pairs=sum(per_step_active), total_pairs=sum(per_step_total),
            per_step_active_pairs=per_step_active, per_step_total_pairs=per_step_total,
            step_inputs=self.step_inputs if self.record_inputs else None,
            step_routes=self.step_routes if self.record_routes else None,
            gpu_seconds=gpu_seconds,
            similarity=(similarity_from_sums(self.sim_sums.cpu().numpy(), self.n)
                        if self.track_similarity and cfg.num_steps > 1 else None))

    def run(self) -> RunResult:
        self.launch()
        return self.finish()


def run_sampling(model: ToyModel, x0: ActivationBlock, strategy: Strategy,
                 policies: PolicyConfig, cluster: ClusterConfig, seed: int, *,
                 record_inputs: bool = False, record_routes: bool = False,
                 track_similarity: bool = False) -> RunResult:
    """Execute a full sampling run on the GPU (schedules.py:493-501).
    track_similarity: step_similarity of the run's own MoE inputs and routes,
    reduced on the device as it runs (RunResult.similarity)."""
    runner = DeviceRunner(model, x0, strategy, policies, cluster, seed,
                          record_inputs=record_inputs, record_routes=record_routes,
                          track_similarity=track_similarity)
    return runner.run()
