"""Peer-memory ghost exchange: producers store straight into their
neighbours' ghost-target rows (NVLink / NVSwitch peer stores between GPUs,
CUDA IPC mappings between processes), so an epoch -- producer, put, gated
epoch kernel, reductions, Adam -- is a fixed sequence of kernels with no
host synchronisation and no NCCL call, captured as ONE CUDA graph.

This replaces the reference's pickled GhostMessage queues (runtime/driver.py:
150-201, worker.py:170-228) for the one-process-per-GPU backend; the message
content is the same (velocity, anchor-normalised pressure on masters,
worker.py:24-46), it just lands in the receiver's target rows directly.

Per rank, one library-allocated block (`fr_ipc_alloc`) holds three monotonic
u32 sync words and the ghost-target rows of every ghost set:

  ready   sources release-add 1 after their rows landed; the epoch kernel's
          ghost sets wait for ready >= rounds * incoming edges (in-kernel,
          fr_epoch_gate.gate_round), bounded by exchange_timeout
  epochs  the rank adds 1 after every epoch kernel (its targets are free);
          a source stores round k's rows for epoch e only once the
          destination's `epochs` reached e (write-after-read guard)
  round   exchange rounds so far (this rank's own counter)

All counters start at 0 in every rank and advance identically, so the
protocol needs no host-side bookkeeping.  See include/flowrec_b200.h.
"""

import ctypes as C

import numpy as np
import torch

from .. import _lib as X

SYNC_BYTES = 256
READY, EPOCHS, ROUND = 0, 4, 8
_ALIGN = 256


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (zero-copy)."""

    _TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int32: "<i4"}

    def __init__(self, ptr, shape, dtype):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": self._TYPESTR[dtype],
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_view(ptr, shape, dtype, device):
    return torch.as_tensor(_CudaArray(ptr, shape, dtype), device=device)


def block_layout(ws, esz, derivatives=False):
    """Byte layout of a rank's block: {(kind, "tu"|"tp"|"tdu"): (offset, shape)}
    and the total size.  Target rows of a kind are concatenated in ghost-index
    order, as DeviceObjective groups them (objective.py:115-141)."""
    nv, nin = ws.regime.n_vel, ws.regime.n_inputs
    counts = {}
    for g in ws.datasets.ghosts:
        counts[g.kind] = counts.get(g.kind, 0) + g.points.shape[0]
    layout = {}
    off = SYNC_BYTES
    for kind in ("spatial", "temporal"):
        n = counts.get(kind, 0)
        if not n:
            continue
        for name, shape in (("tu", (n, nv)), ("tp", (n,))) + ((("tdu", (n, nin, nv)),) if derivatives else ()):
            layout[(kind, name)] = (off, shape)
            off += -(-int(np.prod(shape)) * esz // _ALIGN) * _ALIGN
    return layout, off


def ghost_offsets(ws, layout, esz):
    """ghost index -> byte offsets (u, p, du or -1) and point count of its rows."""
    nv, nin = ws.regime.n_vel, ws.regime.n_inputs
    row = {"spatial": 0, "temporal": 0}
    out = {}
    for gi, g in enumerate(ws.datasets.ghosts):
        n, r = g.points.shape[0], row[g.kind]
        du = layout.get((g.kind, "tdu"))
        out[gi] = (layout[(g.kind, "tu")][0] + r * nv * esz, layout[(g.kind, "tp")][0] + r * esz,
                   du[0] + r * nin * nv * esz if du else -1, n)
        row[g.kind] += n
    return out


class IpcBlock:
    """One rank's peer-visible block: sync words + ghost-target rows per kind.

    `alloc(kind, name, shape)` is the DeviceObjective target allocator; the
    offsets of every ghost index's rows are then published to the peers."""

    def __init__(self, ws, tdtype, device, derivatives=False):
        esz = torch.tensor([], dtype=tdtype).element_size()
        self.ws = ws
        self.layout, self.bytes = block_layout(ws, esz, derivatives)
        self.tdtype, self.device, self.esz = tdtype, device, esz
        ptr = C.c_void_p()
        handle = C.create_string_buffer(X.IPC_HANDLE_BYTES)
        X.call("fr_ipc_alloc", self.bytes, C.byref(ptr), handle)
        self.ptr = int(ptr.value)
        self.handle = handle.raw
        words = device_view(self.ptr, (SYNC_BYTES // 4,), torch.int32, device)
        self.ready, self.epochs, self.round = words[0:1], words[1:2], words[2:3]

    def alloc(self, kind, name, shape):
        off, lshape = self.layout[(kind, name)]
        if tuple(lshape) != tuple(shape):
            raise ValueError(f"ghost target {kind}/{name}: layout {lshape} != requested {shape}")
        return device_view(self.ptr + off, shape, self.tdtype, self.device)

    def target_offsets(self, objective=None):
        """ghost index -> byte offsets (u, p, du or -1) of its rows in this block
        (checked against the objective's own grouping when given)."""
        out = ghost_offsets(self.ws, self.layout, self.esz)
        if objective is not None:
            for gi, (kind, row, n) in objective.ghost_slices.items():
                assert out[gi][0] == self.layout[(kind, "tu")][0] + row * objective.regime.n_vel * self.esz
        return out

    def free(self):
        if self.ptr:
            X.call("fr_ipc_free", C.c_void_p(self.ptr))
            self.ptr = 0


def open_peer(handle):
    ptr = C.c_void_p()
    X.call("fr_ipc_open", C.create_string_buffer(handle, X.IPC_HANDLE_BYTES), C.byref(ptr))
    return int(ptr.value)


def edge_table(edges, dest_info, derivatives=False, rank=None):
    """Plain-tuple form of one source rank's fr_ghost_edge structs (host
    logic only; tested on CPU).

    edges: worker.edges / outgoing_layout(ws)[0] -- (edge, y_row, n,
    anchor_row) in the reference's route order (destination, ghost index;
    driver.py:83-91).  dest_info: dest rank -> (block base address as seen by
    this process, ghost_offsets of the destination).  Returns
    [(y_row, anchor_row, n, u, p, du, ready, epochs)]."""
    if len(edges) > X.MAX_GHOST_EDGES:
        raise ValueError(f"rank {rank} has {len(edges)} outgoing edges (max {X.MAX_GHOST_EDGES})")
    out = []
    for edge, off, n, anc_off in edges:
        base, offsets = dest_info[edge.dest]
        u_off, p_off, du_off, n_dest = offsets[edge.ghost_index]
        if n_dest != n:
            raise ValueError(f"edge {rank}->{edge.dest}[{edge.ghost_index}]: {n} points, destination has {n_dest}")
        out.append((off, -1 if anc_off is None else anc_off, n, base + u_off, base + p_off,
                    base + du_off if (du_off >= 0 and derivatives) else None, base + READY, base + EPOCHS))
    return out


def build_edges(worker, dest_info):
    """fr_ghost_edge array of one source rank (see edge_table)."""
    rows = edge_table(worker.edges, dest_info, worker.send_derivatives, worker.rank)
    arr = (X.GhostEdge * max(1, len(rows)))()
    for k, (y_row, anc, n, u, p, du, ready, epochs) in enumerate(rows):
        e = arr[k]
        e.y_row, e.anchor_row, e.n = y_row, anc, n
        e.u, e.p, e.du, e.ready, e.epochs = u, p, du, ready, epochs
    return arr


class PeerRank:
    """Per-rank enqueue logic of the peer-memory exchange (used one rank per
    process by DistributedTrainer(transport="ipc") and all ranks in one
    process by LocalTrainer(transport="peer"))."""

    def __init__(self, worker, block, timeout_s):
        self.w, self.block = worker, block
        self.timeout_ms = max(1, min(int(round(float(timeout_s) * 1000.0)), 2**32 - 1))
        self.n_in = len(worker.ws.datasets.ghosts)
        self.edges = None
        self.n_edges = len(worker.edges)
        self.gate = None
        if worker.objective.ghost:
            g = worker.objective.make_gate(block.ready, worker.flags, timeout_s)
            g.gate_round, g.gate_mult = block.round.data_ptr(), self.n_in
            self.gate = g

    def connect(self, dest_info):
        self.edges = build_edges(self.w, dest_info)

    def put(self, stream=None):
        """Producer forward + stores into every destination + round counter."""
        w = self.w
        w.produce(stream)
        st = X.stream_ptr(stream)
        if self.n_edges:
            X.call("fr_ghost_put", w.plan.h, X.ptr(w.out_y), X.ptr(w.out_jet), self.n_edges, self.edges,
                   C.c_void_p(self.block.epochs.data_ptr()), self.timeout_ms, X.ptr(w.flags), st)
        X.call("fr_counter_add", C.c_void_p(self.block.round.data_ptr()), 1, st)
        w.objective.mark_targets_set()

    def step(self, exchanged, stream=None):
        """The epoch (gated on this round's arrivals when it exchanged), then
        publish that this rank's targets are free again."""
        w = self.w
        st = X.stream_ptr(stream)
        w.enqueue_epoch(stream, gate=self.gate if exchanged else None,
                        before_update=lambda: X.call("fr_counter_add", C.c_void_p(self.block.epochs.data_ptr()),
                                                     1, st))
