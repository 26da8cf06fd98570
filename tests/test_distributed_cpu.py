"""Multi-process host logic of the NCCL path, on CPU with gloo (world 2 and 8):
every rank posts its ghost round with `post_exchange` over the routes of
`p2p_routes`, and each ghost-target slot must receive exactly the message its
reference route names (source rank, destination ghost index, point count)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, tag, port, q):
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from cases import training_plan
        from conftest import GOLDEN
        from paper_2602_15883_b200.runtime import p2p_routes, post_exchange

        golden = np.load(GOLDEN)
        _, plan = training_plan(tag, golden)
        sends, recvs = p2p_routes(plan, rank)
        nv = plan.regime.n_vel
        # payload encodes (source, destination ghost index, row)
        send_bufs = []
        for dest, k, n in sends:
            gi = plan.worker_specs[rank].outgoing[k].ghost_index
            code = 1000.0 * rank + 10.0 * gi
            u = torch.full((n, nv), code) + torch.arange(n, dtype=torch.float32)[:, None]
            p = -torch.full((n,), code)
            send_bufs.append((u, p))
        recv_bufs = {gi: (torch.zeros((n, nv)), torch.zeros(n)) for _, gi, n in recvs}
        for w in post_exchange(sends, recvs, send_bufs, recv_bufs):
            w.wait()
        ok = True
        for src, gi, n in recvs:
            u, p = recv_bufs[gi]
            code = 1000.0 * src + 10.0 * gi
            ok &= bool(torch.all(u[:, 0] == code + torch.arange(n, dtype=torch.float32)))
            ok &= bool(torch.all(p == -code))
        q.put((rank, ok, len(sends), len(recvs)))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, traceback.format_exc(), 0, 0))


@pytest.mark.parametrize("tag,world", [("p2", 2), ("t2", 2), ("p8", 8)])
def test_ghost_exchange_routes_over_gloo(tag, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tests_dir = os.path.dirname(os.path.abspath(__file__))
    old = os.environ.get("PYTHONPATH", "")
    os.environ["PYTHONPATH"] = os.pathsep.join([tests_dir, os.path.dirname(tests_dir), old])
    procs = [ctx.Process(target=_worker, args=(r, world, tag, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    os.environ["PYTHONPATH"] = old
    for rank, ok, ns, nr in results:
        assert ok is True, (rank, ok)
        assert ns == nr  # every neighbour relation is bidirectional


def _peer_worker(rank, world, tag, port, q):
    """Host logic of the peer-memory transport: every rank publishes its block
    layout (torch.distributed, as DistributedTrainer(transport="ipc") does with
    the real IPC handles), then builds its fr_ghost_edge table against fake
    peer base addresses; each edge must land exactly on the destination's rows
    of the ghost set its route names."""
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from cases import training_plan
        from conftest import GOLDEN
        from paper_2602_15883_b200.runtime.peer import EPOCHS, READY, block_layout, edge_table, ghost_offsets
        from paper_2602_15883_b200.runtime.worker import outgoing_layout

        golden = np.load(GOLDEN)
        _, plan = training_plan(tag, golden)
        ws = plan.worker_specs[rank]
        layout, nbytes = block_layout(ws, 4, derivatives=True)
        table = [None] * world
        dist.all_gather_object(table, (rank, f"handle-{rank}".encode(), ghost_offsets(ws, layout, 4), nbytes))
        base = {r: (r + 1) << 32 for r in range(world)}
        info = {r: (base[r], offs) for r, _, offs, _ in table}
        edges, _, rows = outgoing_layout(ws)
        tab = edge_table(edges, info, derivatives=True, rank=rank)
        ok = len(tab) == len(ws.outgoing)
        claims = []
        for (edge, y_row, n, anc), (yr, ar, n2, u, p, du, ready, ep) in zip(edges, tab):
            d = plan.worker_specs[edge.dest]
            g = d.datasets.ghosts[edge.ghost_index]
            ok &= g.neighbor == rank and g.points.shape[0] == n == n2 and yr == y_row
            ok &= (ar == -1) == (not ws.normalize_outgoing)
            ok &= ready == base[edge.dest] + READY and ep == base[edge.dest] + EPOCHS
            dl, dbytes = block_layout(d, 4, derivatives=True)
            uo = u - base[edge.dest]
            ok &= uo == ghost_offsets(d, dl, 4)[edge.ghost_index][0] and 0 < uo < dbytes
            ok &= du is not None and p - base[edge.dest] < dbytes
            claims.append((edge.dest, edge.ghost_index))
        got = [None] * world
        dist.all_gather_object(got, claims)
        # every ghost set of every rank is written by exactly one source
        flat = sorted(c for cl in got for c in cl)
        expect = sorted((r, gi) for r in range(world) for gi in range(len(plan.worker_specs[r].datasets.ghosts)))
        ok &= flat == expect
        q.put((rank, bool(ok), len(tab), rows))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, traceback.format_exc(), 0, 0))


@pytest.mark.parametrize("tag,world", [("t2", 2), ("p8", 8), ("d3", 8)])
def test_peer_transport_edge_tables_over_gloo(tag, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tests_dir = os.path.dirname(os.path.abspath(__file__))
    old = os.environ.get("PYTHONPATH", "")
    os.environ["PYTHONPATH"] = os.pathsep.join([tests_dir, os.path.dirname(tests_dir), old])
    procs = [ctx.Process(target=_peer_worker, args=(r, world, tag, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    os.environ["PYTHONPATH"] = old
    for rank, ok, n_edges, rows in results:
        assert ok is True, (rank, ok)
        assert n_edges > 0 and rows >= n_edges
