"""Training driver: plan assembly and the GPU epoch loops.

Mirrors pkg/src/flowrec/runtime/driver.py:43-283.  Backends:

  "serial" / "cuda"  every rank in this process on the current GPU (the
                     reference's serial backend, :127-144).  The exchange is
                     device-to-device: each producer packs straight into its
                     destination's ghost-target rows.  After an eager first
                     epoch the loop is replayed from CUDA graphs (one with the
                     exchange, one without), so an epoch costs one graph launch.
  "distributed"      this process is one rank of an initialised
                     torch.distributed group (one process per GPU, launched by
                     torchrun); ghost messages move by NCCL point-to-point
                     straight into the receiver's ghost-target buffers.
  "process"          spawns one process per rank, one GPU each (needs at least
                     as many GPUs as ranks) and runs "distributed" in each.

Semantics kept: the exchange happens before the step of epoch e with the
parameters after epoch e-1, including e = 0 (:133-142); history rows are the
pre-update unweighted parts; masters normalise every outgoing pressure.
"""

import ctypes as C
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from .. import _lib as X
from ..decomposition import identify_masters
from ..network import ExpertConfig, ExpertParams
from ..physics import FlowRegime
from .worker import DeadlockError, OutgoingEdge, RankWorker, TrainConfig, WorkerSpec, derive_param_seed


class RankFailure(RuntimeError):
    pass


@dataclass(frozen=True)
class TrainingPlan:
    regime: FlowRegime
    subdomains: tuple
    masters: frozenset
    expert_config: ExpertConfig
    train_config: TrainConfig
    worker_specs: tuple

    @property
    def n_ranks(self):
        return len(self.worker_specs)


@dataclass
class TrainResult:
    params: dict
    history: dict
    epoch_times: dict
    exchange_log: dict
    wall_time_s: float = 0.0

    def median_epoch_time(self):
        """Median over epochs of the slowest rank's epoch duration (:65-68)."""
        stacked = np.stack([self.epoch_times[r] for r in sorted(self.epoch_times)])
        return float(np.median(np.max(stacked, axis=0)))


def build_plan(subdomains, datasets, expert_config: ExpertConfig, train_config: TrainConfig) -> TrainingPlan:
    """Roles, effective weights and message routes (driver.py:71-121)."""
    regime = subdomains[0].domain.regime
    anchored = train_config.pressure_coupling == "anchored_master"
    masters = identify_masters(subdomains, train_config.anchor)
    if anchored and subdomains[0].time_splits > 1 and not train_config.weights.ghost_p_time > 0:
        raise ValueError("temporal ghost pressure weight must be positive when the domain is split in time")
    outgoing = {s.rank_index: [] for s in subdomains}
    for s in subdomains:
        ds = datasets[s.rank_index]
        if len(ds.ghosts) != len(s.ghosts):
            raise ValueError(f"rank {s.rank_index}: datasets do not match the partition")
        for gi, g in enumerate(ds.ghosts):
            outgoing[g.neighbor].append(OutgoingEdge(s.rank_index, gi, g.kind, g.points))
    specs = []
    for s in subdomains:
        master = anchored and s.rank_index in masters
        w = train_config.weights.as_master() if master else train_config.weights
        specs.append(WorkerSpec(
            rank=s.rank_index, role="master" if master else "slave", spec=s, regime=regime,
            expert_config=expert_config, train_config=train_config, datasets=datasets[s.rank_index],
            effective_weights=w, outgoing=tuple(outgoing[s.rank_index]),
            param_seed=derive_param_seed(train_config.seed, s.rank_index), normalize_outgoing=master,
        ))
    return TrainingPlan(regime, tuple(subdomains), masters, expert_config, train_config, tuple(specs))


# -- in-process (single GPU, all ranks) ---------------------------------------------


def _free_sms_without_extra_wave(plan, ws, most=2):
    """SMs the overlapped exchange may keep free (up to `most`) without adding
    a wave of tiles to this rank's persistent epoch kernel; 0 if even one
    would (the exchange then runs in stream order on the full grid)."""
    from ..engine import get_plan

    tc = plan.train_config
    ep = get_plan(plan.expert_config, plan.regime.kind, plan.regime.reynolds, "float32", tc.math)
    d = ws.datasets
    per_kind = {}
    for g in d.ghosts:
        per_kind[g.kind] = per_kind.get(g.kind, 0) + g.points.shape[0]
    sets = ([d.n_obs] if d.n_obs else []) + [per_kind[k] for k in ("spatial", "temporal") if k in per_kind]
    n_sets = (C.c_longlong * 3)(*(sets + [0] * 3)[:3])
    wsp = X.Workspace()
    X.call("fr_epoch_workspace", ep.h, d.n_colloc, n_sets, len(sets), C.byref(wsp))
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    waves = -(-wsp.tiles // sms)
    for r in range(most, 0, -1):
        if -(-wsp.tiles // (sms - r)) == waves:
            return r
    return 0


def _overlap_max_ctas(reserve_sms):
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return max(1, sms - int(reserve_sms))


class LocalTrainer:
    """All ranks of a plan resident on one GPU with a device-to-device exchange.

    overlap=True runs the exchange the way the one-process-per-GPU trainer
    does: the packs into the destinations' target rows go on a transport
    stream that publishes each rank's gate word, and the epoch kernels start
    at once, their ghost heads waiting in-kernel (fr_epoch_fwd_bwd_gated).
    `signal_delay_ns` holds every gate back that long (tests use it to prove
    the in-kernel wait, not stream order, protects the ghost heads)."""

    def __init__(self, plan: TrainingPlan, dtype="float32", epochs=None, overlap=False, reserve_sms=None,
                 signal_delay_ns=0, exchange_timeout=600.0, transport="device"):
        """transport="device": packs write the destinations' target rows in
        stream order (or on a side stream with overlap=True); "peer": every
        rank runs the peer-memory protocol of the one-process-per-GPU trainer
        (runtime/peer.py: fr_ghost_put into the destination's IPC block, the
        ready / epochs counters, the counter-gated epoch kernel), enqueued on
        one stream so each wait is already satisfied when it is reached."""
        if transport not in ("device", "peer"):
            raise ValueError(f"unknown transport {transport!r} (use 'device' or 'peer')")
        if transport == "peer" and overlap:
            raise ValueError("the in-process peer transport runs stream-ordered (overlap=False)")
        self.plan = plan
        self.transport = transport
        self.exchange_timeout = float(exchange_timeout)
        self.overlap = bool(overlap)
        self.signal_delay_ns = int(signal_delay_ns)
        if reserve_sms is None:
            reserve_sms = 2 if self.overlap else 0
        max_ctas = _overlap_max_ctas(reserve_sms) if reserve_sms else 0
        self.blocks = {}
        if transport == "peer":
            from .peer import IpcBlock

            dev = torch.device("cuda", torch.cuda.current_device())
            tdt = torch.float32 if dtype in ("float32", "f32") else torch.float64
            self.blocks = {ws.rank: IpcBlock(ws, tdt, dev, plan.train_config.ghost_derivative_weight > 0)
                           for ws in plan.worker_specs}
        self.workers = {ws.rank: RankWorker(ws, dtype=dtype, epochs=epochs, max_ctas=max_ctas,
                                            target_alloc=self.blocks[ws.rank].alloc if self.blocks else None)
                        for ws in plan.worker_specs}
        self.order = sorted(self.workers)
        if transport == "peer":
            from .peer import PeerRank

            self.peers = {r: PeerRank(self.workers[r], self.blocks[r], self.exchange_timeout) for r in self.order}
            info = {r: (self.blocks[r].ptr, self.blocks[r].target_offsets(self.workers[r].objective))
                    for r in self.order}
            for r in self.order:
                self.peers[r].connect(info)
        if self.overlap:
            self.comm = torch.cuda.Stream()
            self.gates = torch.zeros(len(self.order), dtype=torch.int32, device="cuda")
            self.gate_args = {r: self.workers[r].objective.make_gate(self.gates[i], self.workers[r].flags,
                                                                     self.exchange_timeout)
                              for i, r in enumerate(self.order)}
        self.routes = []
        for r in self.order:
            w = self.workers[r]
            for k, (edge, _, _, _) in enumerate(w.edges):
                dobj = self.workers[edge.dest].objective
                tu, tp = dobj.target_slice(edge.ghost_index)
                self.routes.append((w, k, tu, tp, dobj.target_du_slice(edge.ghost_index)))
        self.graphs = {}
        self._ran_eager = False

    def close(self):
        """Free the peer transport's blocks (after the device is idle)."""
        if self.blocks:
            torch.cuda.synchronize()
            for b in self.blocks.values():
                b.free()
            self.blocks = {}

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def enqueue_exchange(self):
        for r in self.order:
            self.workers[r].produce()
        for w, k, tu, tp, tdu in self.routes:
            w.pack_edge(k, tu, tp, out_du=tdu)
        for w in self.workers.values():
            w.objective.mark_targets_set()

    def enqueue_step(self):
        for r in self.order:
            self.workers[r].enqueue_epoch()

    def _enqueue(self, exchange):
        if self.transport == "peer":
            if exchange:
                for r in self.order:
                    self.peers[r].put()
            for r in self.order:
                self.peers[r].step(exchange)
            return
        if exchange and self.overlap:
            self._enqueue_overlapped()
            return
        if exchange:
            self.enqueue_exchange()
        self.enqueue_step()

    def _enqueue_overlapped(self):
        for r in self.order:
            self.workers[r].produce()
        self.gates.zero_()
        cur = torch.cuda.current_stream()
        self.comm.wait_stream(cur)
        with torch.cuda.stream(self.comm):
            for w, k, tu, tp, tdu in self.routes:
                w.pack_edge(k, tu, tp, stream=self.comm, out_du=tdu)
            for i, r in enumerate(self.order):
                X.call("fr_signal", C.c_void_p(self.gates[i].data_ptr()), 1, self.signal_delay_ns,
                       X.stream_ptr(self.comm))
        for w in self.workers.values():
            w.objective.mark_targets_set()
        for r in self.order:
            self.workers[r].enqueue_epoch(gate=self.gate_args[r] if self.workers[r].objective.ghost else None)
        cur.wait_stream(self.comm)

    def _graph(self, exchange, epochs=1):
        """CUDA graph of `epochs` consecutive epochs, the first with the
        exchange iff `exchange` (a whole comm_interval block is one replay)."""
        key = (exchange, epochs)
        g = self.graphs.get(key)
        if g is None:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(epochs):
                    self._enqueue(exchange and i == 0)
            self.graphs[key] = g
        return g

    def check_flags(self):
        for w in self.workers.values():
            w.check_flags()

    def log_exchange(self, e):
        for w in self.workers.values():
            w.exchange_log.append((e, sorted(w.expected_messages)))

    def run(self, epochs, start=0, use_graphs=True, record_times=True, unroll=False):
        """Train `epochs` epochs; returns per-epoch device times (s).

        unroll=True (needs record_times=False) replays each whole
        comm_interval block -- the exchange epoch and the comm_interval - 1
        epochs that reuse its targets -- as ONE graph."""
        comm = self.plan.train_config.comm_interval
        if unroll and record_times:
            raise ValueError("unrolled graph blocks are timed as a whole; use record_times=False")
        events = []
        e, end = start, start + epochs
        while e < end:
            exchange = e % comm == 0
            block = 1
            if unroll and use_graphs and self._ran_eager and exchange and e + comm <= end:
                block = comm
            if record_times:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                events.append(ev)
            # the trainer's first epoch runs eagerly (it also initialises every
            # lazily set attribute); later epochs replay captured graphs of the
            # same work
            if use_graphs and self._ran_eager:
                # a replay bypasses enqueue_epoch's capacity check: the optimiser
                # kernel indexes the schedule / history rows by its step counter
                for w in self.workers.values():
                    if w.epochs_done + block > w.capacity:
                        raise RuntimeError("history capacity exhausted; construct the trainer with more epochs")
                self._graph(exchange, block).replay()
            else:
                self._enqueue(exchange)
                self._ran_eager = True
            if exchange:
                self.log_exchange(e)
            for w in self.workers.values():
                w.epochs_done += block
            e += block
        if not record_times:
            return None  # asynchronous: caller synchronises and calls check_flags()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        events.append(ev)
        torch.cuda.synchronize()
        self.check_flags()
        times = np.array([a.elapsed_time(b) * 1e-3 for a, b in zip(events[:-1], events[1:])])
        for w in self.workers.values():
            w.epoch_times.extend(times.tolist())
        return times


def _train_local(plan, dtype, use_graphs, exchange_timeout=600.0):
    t0 = time.perf_counter()
    trainer = LocalTrainer(plan, dtype=dtype, exchange_timeout=exchange_timeout)
    trainer.run(plan.train_config.epochs, use_graphs=use_graphs)
    return _collect(plan, {r: w.export() for r, w in trainer.workers.items()}, time.perf_counter() - t0)


# -- one process per GPU -------------------------------------------------------------


def p2p_routes(plan: TrainingPlan, rank: int):
    """(sends, recvs) of one rank: sends [(dest, edge_index, n)], recvs
    [(source, ghost_index, n)], both sorted by (peer, ghost index) (:83-91)."""
    ws = plan.worker_specs[rank]
    sends = [(e.dest, k, e.points.shape[0]) for k, e in enumerate(ws.outgoing)]
    recvs = [(g.neighbor, gi, g.points.shape[0]) for gi, g in enumerate(ws.datasets.ghosts)]
    return sends, recvs


def post_exchange(sends, recvs, send_bufs, recv_bufs, group=None):
    """Issue every send/recv of one round as a single batched P2P group.

    send_bufs[k] / recv_bufs[gi] are (u, p) tensor pairs, or (u, p, du) with
    the derivative-coupling extension.  Returns the work
    handles; waiting on them orders the caller's stream after the transfers."""
    import torch.distributed as dist

    ops = []
    for dest, k, _ in sends:
        ops += [dist.P2POp(dist.isend, t, dest, group) for t in send_bufs[k]]
    for src, gi, _ in recvs:
        ops += [dist.P2POp(dist.irecv, t, src, group) for t in recv_bufs[gi]]
    return dist.batch_isend_irecv(ops) if ops else []


class FrNcclTransport:
    """The library's own exchange transport (fr_nccl_init / fr_exchange, the C
    ABI of SURVEY 8b): rank 0 makes the NCCL unique id, torch.distributed
    broadcasts it once, and every exchange round is one grouped
    ncclSend/ncclRecv set enqueued on the current stream."""

    def __init__(self, dtype):
        import torch.distributed as dist

        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            X.call("fr_nccl_get_unique_id", uid)
        box = [uid.raw]
        dist.broadcast_object_list(box, src=0)
        uid = C.create_string_buffer(box[0], 128)
        self.comm = C.c_void_p()
        X.call("fr_nccl_init", uid, self.world, self.rank, C.byref(self.comm))
        self.dtype = X.F32 if dtype == "float32" else X.F64

    def __call__(self, sends, recvs, send_bufs, recv_bufs, group=None):
        sp, sb, sc, rp, rb, rc = [], [], [], [], [], []
        for dest, k, _ in sends:
            for t in send_bufs[k]:
                sp.append(dest), sb.append(t.data_ptr()), sc.append(t.numel())
        for src, gi, _ in recvs:
            for t in recv_bufs[gi]:
                rp.append(src), rb.append(t.data_ptr()), rc.append(t.numel())
        arr = lambda ty, v: (ty * max(len(v), 1))(*v)  # noqa: E731
        X.call("fr_exchange", self.comm, len(sp), arr(C.c_int, sp), arr(C.c_void_p, sb), arr(C.c_longlong, sc),
               len(rp), arr(C.c_int, rp), arr(C.c_void_p, rb), arr(C.c_longlong, rc), self.dtype, X.stream_ptr())
        return []  # enqueued on the current stream: nothing to wait for

    def close(self):
        if self.comm:
            X.call("fr_nccl_destroy", self.comm)
            self.comm = C.c_void_p()


def _peer_access_everywhere(n_ranks):
    """True when every visible GPU pair used by an n_ranks job (one per GPU,
    or all ranks on one GPU) can access each other's memory."""
    n_dev = torch.cuda.device_count()
    devs = range(min(n_dev, n_ranks))
    return all(a == b or torch.cuda.can_device_access_peer(a, b) for a in devs for b in devs)


class DistributedTrainer:
    """This process's rank of a torch.distributed group (one process per GPU).

    transport="ipc" (default): the peer-memory exchange of runtime/peer.py --
    the producer's put kernel stores the ghost rows straight into the
    neighbours' target blocks over NVLink (CUDA IPC mappings), arrivals are
    counted in the receiver's `ready` word and its epoch kernel's ghost sets
    wait on that count in-kernel; no NCCL call and no host synchronisation
    per epoch, so every epoch after the first is ONE CUDA graph replay.
    torch.distributed is used once, to exchange the IPC handles.

    transport="torch" / "fr_nccl" (NCCL point-to-point, enqueued eagerly):
    overlap=True (default for the fused small-width kernel): the ghost
    transfer is overlapped with the interior work.  The producer (value
    forward of the neighbours' ghost points) and the pack run on the compute
    stream (~20 us); the NCCL send/recv group then runs on a transport stream
    which, once the receives have landed, sets this rank's gate word
    (fr_signal).  The epoch kernel is launched at once with its persistent grid
    capped `reserve_sms` below the SM count, so NCCL's kernels have an SM to run
    on; every CTA walks its PDE and observation tiles first and only its ghost
    tiles wait on the gate.  By default the reserve is the largest of 2, 1 SMs
    that does not add a wave of tiles to the kernel (P=8: 1319 tiles, 147 CTAs
    keep 9 per CTA where 146 would need 10); if even one SM would, the exchange
    runs in stream order on the full grid.  The first exchange always runs in
    stream order (it also brings up the NCCL connections, which may
    synchronise the device)."""

    def __init__(self, plan: TrainingPlan, rank=None, dtype="float32", epochs=None, overlap=True, reserve_sms=None,
                 transport="ipc", exchange_timeout=600.0):
        import torch.distributed as dist

        if transport not in ("torch", "fr_nccl", "ipc"):
            raise ValueError(f"unknown transport {transport!r} (use 'ipc', 'torch' or 'fr_nccl')")

        self.plan = plan
        self.transport = transport
        self.rank = dist.get_rank() if rank is None else rank
        if dist.get_world_size() != plan.n_ranks:
            raise ValueError(f"world size {dist.get_world_size()} != plan ranks {plan.n_ranks}")
        ws = plan.worker_specs[self.rank]
        self.graphs = {}
        self.launches_per_epoch = {}  # library kernels in each captured epoch graph
        self._ran_eager = False
        if transport == "ipc" and not _peer_access_everywhere(plan.n_ranks):
            # the peer-memory transport needs every pair of this node's GPUs to
            # reach each other's memory (NVLink / NVSwitch); otherwise NCCL P2P
            import warnings

            warnings.warn("GPUs without peer access: the ghost exchange falls back to NCCL point-to-point")
            transport = self.transport = "torch"
        if transport == "ipc":
            self._init_ipc(plan, ws, dtype, epochs, exchange_timeout)
            return
        wide = max(plan.expert_config.arch[1:-1], default=0) > 64
        self.overlap = bool(overlap) and not wide and len(ws.datasets.ghosts) > 0
        max_ctas = 0
        if self.overlap:
            if reserve_sms is None:
                reserve_sms = _free_sms_without_extra_wave(plan, ws)
            if reserve_sms > 0:
                max_ctas = _overlap_max_ctas(reserve_sms)
            else:
                self.overlap = False  # reserving an SM would cost a whole extra tile wave
        self.worker = w = RankWorker(ws, dtype=dtype, epochs=epochs, max_ctas=max_ctas)
        self.sends, self.recvs = p2p_routes(plan, self.rank)
        nv, T, dev = plan.regime.n_vel, w.plan.tdtype, w.plan.device
        nin = plan.regime.n_inputs
        self.send_bufs = [(torch.empty((n, nv), dtype=T, device=dev), torch.empty(n, dtype=T, device=dev))
                          + ((torch.empty((n, nin, nv), dtype=T, device=dev),) if w.send_derivatives else ())
                          for _, _, n in self.sends]
        self.recv_bufs = {gi: w.objective.target_slice(gi)
                          + ((w.objective.target_du_slice(gi),) if w.send_derivatives else ())
                          for _, gi, _ in self.recvs}
        self._connected = False
        # exchange rounds: torch.distributed batched P2P, or the library's own
        # NCCL transport (fr_exchange)
        self._post = FrNcclTransport(dtype) if transport == "fr_nccl" else None
        if self.overlap:
            self.comm = torch.cuda.Stream()
            self.gate_word = torch.zeros(1, dtype=torch.int32, device=dev)
            # the in-kernel wait is bounded by the reference's exchange timeout
            # (driver.py:150-181): a lost peer -> FLAG_EXCHANGE_TIMEOUT -> DeadlockError
            self.gate = w.objective.make_gate(self.gate_word, w.flags, exchange_timeout)

    def _init_ipc(self, plan, ws, dtype, epochs, exchange_timeout):
        """Peer-memory transport (runtime/peer.py): the neighbours' target
        blocks are mapped into this process (CUDA IPC, peer access over
        NVLink); every epoch is a fixed kernel sequence, replayed from CUDA
        graphs after the first."""
        import torch.distributed as dist

        from .peer import IpcBlock, PeerRank, open_peer

        self.overlap = False
        dev = torch.device("cuda", torch.cuda.current_device())
        tdt = torch.float32 if dtype in ("float32", "f32") else torch.float64
        self.block = IpcBlock(ws, tdt, dev, plan.train_config.ghost_derivative_weight > 0)
        self.worker = w = RankWorker(ws, dtype=dtype, epochs=epochs, target_alloc=self.block.alloc)
        torch.cuda.synchronize()  # the block is zeroed before any peer can store into it
        mine = (self.rank, self.block.handle, self.block.target_offsets(w.objective))
        table = [None] * plan.n_ranks
        dist.all_gather_object(table, mine)
        self.peer_ptrs = {}
        info = {}
        for r, handle, offsets in table:
            if r in {e.dest for e in ws.outgoing}:
                self.peer_ptrs[r] = open_peer(handle)
                info[r] = (self.peer_ptrs[r], offsets)
        self.peer = PeerRank(w, self.block, exchange_timeout)
        self.peer.connect(info)

    def _enqueue_ipc(self, exchange):
        if exchange:
            self.peer.put()
        self.peer.step(exchange)

    def _ipc_epoch(self, exchange, use_graphs=True):
        if use_graphs and self._ran_eager:
            w = self.worker
            if w.epochs_done + 1 > w.capacity:
                raise RuntimeError("history capacity exhausted; construct the trainer with more epochs")
            g = self.graphs.get(exchange)
            if g is None:
                from .. import _lib as X

                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                k0 = X.kernel_launches()
                with torch.cuda.graph(g):
                    self._enqueue_ipc(exchange)
                self.launches_per_epoch[exchange] = X.kernel_launches() - k0
                self.graphs[exchange] = g
            g.replay()
        else:
            self._enqueue_ipc(exchange)
            self._ran_eager = True

    def close(self):
        """Unmap the peers' blocks (IPC) / destroy the library's communicator.
        This rank's own block is freed by `free()`, once every peer has closed
        (a barrier between the two on every rank)."""
        from .. import _lib as X

        for ptr in getattr(self, "peer_ptrs", {}).values():
            X.call("fr_ipc_close", C.c_void_p(ptr))
        self.peer_ptrs = {}
        if getattr(self, "_post", None) is not None and hasattr(self._post, "close"):
            self._post.close()

    def free(self):
        blk = getattr(self, "block", None)
        if blk is not None:
            torch.cuda.synchronize()
            blk.free()

    def _du(self, k):
        b = self.send_bufs[k]
        return b[2] if len(b) > 2 else None

    def epoch(self, e, use_graphs=True):
        """Exchange (if due) then the fused epoch (overlapped, see the class doc)."""
        w = self.worker
        exchange = e % self.plan.train_config.comm_interval == 0
        if self.transport == "ipc":
            self._ipc_epoch(exchange, use_graphs)
            w.epochs_done += 1
            if exchange:
                w.exchange_log.append((e, sorted(w.expected_messages)))
            return
        cur = torch.cuda.current_stream()
        if exchange and self.overlap and self._connected:
            # producer + pack on the compute stream (~20 us on the full GPU);
            # the NCCL group and the gate signal on the transport stream, on the
            # reserved SM(s), while the epoch kernel walks its interior tiles
            w.produce()
            for k, _ in enumerate(self.sends):
                w.pack_edge(k, *self.send_bufs[k][:2], out_du=self._du(k))
            self.gate_word.zero_()
            ready = torch.cuda.Event()
            ready.record(cur)
            w.objective.mark_targets_set()
            self.comm.wait_event(ready)
            with torch.cuda.stream(self.comm):
                for wk in (self._post or post_exchange)(self.sends, self.recvs, self.send_bufs, self.recv_bufs):
                    wk.wait()  # transport stream waits for the transfers
                X.call("fr_signal", C.c_void_p(self.gate_word.data_ptr()), 1, 0, X.stream_ptr(self.comm))
            # the next round reuses the send buffers and targets
            w.enqueue_epoch(gate=self.gate, before_update=lambda: cur.wait_stream(self.comm))
        else:
            if exchange:
                w.produce()
                for k, _ in enumerate(self.sends):
                    w.pack_edge(k, *self.send_bufs[k][:2], out_du=self._du(k))
                for wk in (self._post or post_exchange)(self.sends, self.recvs, self.send_bufs, self.recv_bufs):
                    wk.wait()  # orders the compute stream after the transfers (no host sync)
                self._connected = True
                w.objective.mark_targets_set()
            w.enqueue_epoch()
        w.epochs_done += 1
        if exchange:
            w.exchange_log.append((e, sorted(w.expected_messages)))

    def run(self, epochs, start=0):
        events = []
        for e in range(start, start + epochs):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            events.append(ev)
            self.epoch(e)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        events.append(ev)
        torch.cuda.synchronize()
        self.worker.check_flags()
        times = [a.elapsed_time(b) * 1e-3 for a, b in zip(events[:-1], events[1:])]
        self.worker.epoch_times.extend(times)
        return times


def _train_distributed(plan, dtype, exchange_timeout=600.0, transport="ipc"):
    import torch.distributed as dist

    t0 = time.perf_counter()
    tr = DistributedTrainer(plan, dtype=dtype, exchange_timeout=exchange_timeout, transport=transport)
    tr.run(plan.train_config.epochs)
    exports = [None] * plan.n_ranks
    dist.all_gather_object(exports, (tr.rank, tr.worker.export()))
    dist.barrier()  # no peer may unmap / free a block another rank still stores into
    tr.close()
    dist.barrier()  # every peer has unmapped this rank's block
    tr.free()
    return _collect(plan, dict(exports), time.perf_counter() - t0)


def _process_entry(local_rank, plan, dtype, port, q, exchange_timeout=600.0):
    import torch.distributed as dist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", rank=local_rank, world_size=plan.n_ranks)
        res = _train_distributed(plan, dtype, exchange_timeout)
        if local_rank == 0:
            q.put(("ok", res))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put(("error", f"rank {local_rank}:\n{traceback.format_exc()}"))


def _train_process(plan, dtype, timeout):
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < plan.n_ranks:
        raise RankFailure(f"backend 'process' needs {plan.n_ranks} GPUs, found {torch.cuda.device_count()}")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_process_entry, args=(r, plan, dtype, port, q, timeout), daemon=True)
             for r in range(plan.n_ranks)]
    for p in procs:
        p.start()
    try:
        status, payload = q.get(timeout=max(timeout, 60.0) * 4)
    except Exception:
        status, payload = "error", "coordinator timed out waiting for rank results"
    finally:
        for p in procs:
            p.join(timeout=30.0)
            if p.is_alive():
                p.terminate()
    if status != "ok":
        raise RankFailure(f"training aborted:\n{payload}")
    return payload


def _collect(plan, exports, wall):
    params, history, times, xlog = {}, {}, {}, {}
    for ws in plan.worker_specs:
        ex = exports[ws.rank]
        params[ws.rank] = ExpertParams(plan.expert_config, np.asarray(ex["flat"]), seed=ex["param_seed"])
        history[ws.rank] = np.asarray(ex["history"])
        times[ws.rank] = np.asarray(ex["epoch_times"])
        xlog[ws.rank] = ex["exchange_log"]
    return TrainResult(params, history, times, xlog, wall_time_s=wall)


def train(plan: TrainingPlan, backend="serial", exchange_timeout=600.0, dtype="float32", use_graphs=True):
    """Run the distributed training loop on the GPU(s)."""
    if not exchange_timeout > 0:
        raise ValueError("exchange timeout must be positive")
    if backend in ("serial", "cuda"):
        return _train_local(plan, dtype, use_graphs, exchange_timeout)
    if backend == "distributed":
        return _train_distributed(plan, dtype, exchange_timeout)
    if backend == "process":
        return _train_process(plan, dtype, exchange_timeout)
    raise ValueError(f"unknown backend {backend!r} (use 'serial', 'cuda', 'distributed' or 'process')")


def train_many(plans, n_workers=1, backend="serial", exchange_timeout=600.0, dtype="float32"):
    """Independent plans (e.g. one per seed): replicas, run one after another."""
    return [train(p, backend=backend, exchange_timeout=exchange_timeout, dtype=dtype) for p in plans]
