"""Peer-memory ghost transport (runtime/peer.py: fr_ipc_alloc blocks,
fr_ghost_put stores into the destination's target rows, ready / epochs
counters, counter-gated epoch kernel) run for every rank in one process on
one stream -- each wait is already satisfied when it is reached, so no kernel
ever waits on another running one -- and compared bit for bit with the
stream-ordered device-to-device trainer; every epoch after the first replays
one CUDA graph."""

import numpy as np
import pytest

from cases import training_plan

pytestmark = pytest.mark.gpu


def _same(a, b):
    for r in a.workers:
        wa, wb = a.workers[r], b.workers[r]
        assert np.array_equal(wa.flat.cpu().numpy(), wb.flat.cpu().numpy()), r
        wa.sync_history()
        wb.sync_history()
        assert np.array_equal(np.array(wa.history)[:, 1:], np.array(wb.history)[:, 1:]), r
        assert wa.exchange_log == wb.exchange_log


@pytest.mark.parametrize("tag", ["t2", "p8", "d3"])
def test_peer_transport_bit_identical(golden, tag):
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = training_plan(tag, golden)
    epochs = plan.train_config.epochs
    a = LocalTrainer(plan)
    a.run(epochs)
    b = LocalTrainer(plan, transport="peer")
    b.run(epochs)
    _same(a, b)
    assert set(b.graphs) == {(True, 1)}  # epochs 1.. replay one captured graph
    for r, blk in b.blocks.items():
        n_in = len(plan.worker_specs[r].datasets.ghosts)
        assert int(blk.epochs.item()) == epochs
        assert int(blk.round.item()) == epochs
        assert int(blk.ready.item()) == epochs * n_in


def test_peer_transport_comm_interval_and_derivatives():
    """comm_interval 3 (targets reused between rounds, unrolled graph blocks)
    with the C^1 extension's derivative targets carried by the put kernel."""
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    pb = fconfig.cylinder2d_problem(n_pde=3000, n_ghost=40, per_snapshot=12, grid_nx=9, snapshots=10,
                                    hidden_layers=3, width=64, activation="tanh", counts=(2, 2), time_splits=2)
    tc = TrainConfig(epochs=7, batch_size=500, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                     comm_interval=3, seed=0, ghost_derivative_weight=0.3)
    plan = build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)
    a = LocalTrainer(plan)
    a.run(7)
    b = LocalTrainer(plan, transport="peer")
    b.run(7, use_graphs=True, record_times=False, unroll=True)
    import torch

    torch.cuda.synchronize()
    b.check_flags()
    _same(a, b)
    assert (True, 3) in b.graphs
    for blk in b.blocks.values():
        assert int(blk.round.item()) == 3 and int(blk.epochs.item()) == 7


def test_peer_put_times_out_when_destination_never_frees(golden):
    """A destination whose `epochs` word never advances: the put kernel gives
    up after the exchange timeout and flags it (DeadlockError on the host)."""
    import ctypes as C

    import torch

    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200.runtime import DeadlockError
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = training_plan("t2", golden)
    tr = LocalTrainer(plan, transport="peer", exchange_timeout=0.02)
    src = tr.peers[0]
    # pretend rank 0 already finished 5 epochs: its put waits for rank 1 to reach 5
    X.call("fr_counter_add", C.c_void_p(tr.blocks[0].epochs.data_ptr()), 5, X.stream_ptr())
    src.put()
    torch.cuda.synchronize()
    with pytest.raises(DeadlockError):
        tr.workers[0].check_flags()


def _ipc_child(handle, q):
    try:
        import ctypes as C

        import torch

        from paper_2602_15883_b200 import _lib as X
        from paper_2602_15883_b200.runtime.peer import READY, open_peer

        torch.cuda.set_device(0)
        base = open_peer(handle)
        X.call("fr_counter_add", C.c_void_p(base + READY), 7, X.stream_ptr())
        torch.cuda.synchronize()
        X.call("fr_ipc_close", C.c_void_p(base))
        q.put("ok")
    except Exception:
        import traceback

        q.put(traceback.format_exc())


def test_ipc_handle_opens_in_another_process():
    """The block a DistributedTrainer publishes is writable from another
    process through its IPC handle (no kernel waits on another here: the child
    adds to the parent's ready word and exits, then the parent reads it)."""
    import torch
    import torch.multiprocessing as mp

    from paper_2602_15883_b200.runtime.peer import IpcBlock

    _, plan = training_plan("t2", __import__("numpy").load(__import__("conftest").GOLDEN))
    blk = IpcBlock(plan.worker_specs[0], torch.float32, torch.device("cuda", 0))
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ipc_child, args=(blk.handle, q))
    p.start()
    msg = q.get(timeout=300)
    p.join(timeout=60)
    assert msg == "ok", msg
    assert int(blk.ready.item()) == 7
    blk.free()


def test_distributed_trainer_ipc_world1(golden):
    """DistributedTrainer(transport='ipc') end to end in a one-rank group
    (handle table over torch.distributed, graph replays) == LocalTrainer."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2602_15883_b200.runtime.driver import DistributedTrainer, LocalTrainer

    _, plan = training_plan("p1", golden)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        tr = DistributedTrainer(plan, transport="ipc")
        tr.run(plan.train_config.epochs)
        assert set(tr.graphs) == {True} and tr.launches_per_epoch[True] > 0
        ref = LocalTrainer(plan)
        ref.run(plan.train_config.epochs)
        assert np.array_equal(tr.worker.flat.cpu().numpy(), ref.workers[0].flat.cpu().numpy())
        tr.worker.sync_history()
        ref.workers[0].sync_history()
        assert np.array_equal(np.array(tr.worker.history)[:, 1:], np.array(ref.workers[0].history)[:, 1:])
        tr.close()
        tr.free()
    finally:
        dist.destroy_process_group()
