"""Overlapped ghost exchange (fr_epoch_fwd_bwd_gated + fr_signal): the epoch
kernel starts before the ghost targets exist and its ghost heads wait in-kernel
on a gate word that the transport stream publishes.  Checked with
the in-process transport, whose packs run on a side stream exactly as the NCCL
receives do in the one-process-per-GPU trainer."""

import numpy as np
import pytest

from cases import training_plan
from conftest import max_rel, rel_l2

pytestmark = pytest.mark.gpu


def _run(plan, epochs, **kw):
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    tr = LocalTrainer(plan, **kw)
    tr.run(epochs)
    out = {}
    for r, w in tr.workers.items():
        w.sync_history()
        out[r] = (w.flat.cpu().numpy(), np.array(w.history))
    return out


@pytest.mark.parametrize("tag", ["t2", "p8"])
def test_overlapped_exchange_bit_identical_to_stream_ordered(golden, tag):
    """Same persistent grid (2 SMs reserved), gate held back 300 us per round:
    identical parameters and history to the stream-ordered exchange, eager
    first epoch and graph replays alike."""
    _, plan = training_plan(tag, golden)
    n = plan.train_config.epochs
    a = _run(plan, n, overlap=False, reserve_sms=2)
    b = _run(plan, n, overlap=True, reserve_sms=2, signal_delay_ns=300_000)
    for r in a:
        assert np.array_equal(a[r][0], b[r][0]), r
        assert np.array_equal(a[r][1][:, 1:], b[r][1][:, 1:]), r


def test_overlapped_training_matches_reference(golden):
    _, plan = training_plan("p8", golden)
    res = _run(plan, plan.train_config.epochs, overlap=True)
    for r, (flat, hist) in res.items():
        assert max_rel(hist[:, 1:6], golden[f"p8/r{r}/history"][:, 1:6]) < 1e-5
        assert rel_l2(flat, golden[f"p8/r{r}/final"]) < 1e-6


def test_gate_timeout_flags_deadlock(golden):
    """A gate that is never published times out inside the kernel, sets the
    exchange-timeout flag and surfaces as DeadlockError (driver.py:161-166)."""
    import torch

    from paper_2602_15883_b200 import _lib as X
    from paper_2602_15883_b200.runtime import DeadlockError, RankWorker

    _, plan = training_plan("t2", golden)
    w = RankWorker(plan.worker_specs[0], max_ctas=8)
    w.objective.mark_targets_set()
    gate_word = torch.zeros(1, dtype=torch.int32, device="cuda")
    gate = w.objective.make_gate(gate_word, w.flags, timeout_s=0.02)
    w.enqueue_epoch(gate=gate)
    torch.cuda.synchronize()
    assert int(w.flags.item()) & X.FLAG_EXCHANGE_TIMEOUT
    with pytest.raises(DeadlockError):
        w.check_flags()


@pytest.mark.parametrize("overlap", [False, True])
def test_unrolled_comm_interval_blocks_bit_identical(overlap):
    """comm_interval = 3: replaying each exchange block (1 exchange epoch +
    2 epochs on the same targets) as one CUDA graph changes nothing."""
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    pb = fconfig.cylinder2d_problem(n_pde=2000, n_ghost=40, per_snapshot=12, grid_nx=9, snapshots=10,
                                    hidden_layers=2, width=32, activation="tanh", counts=(2, 1), time_splits=2)
    tc = TrainConfig(epochs=8, batch_size=500, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                     lr_factor=0.5, lr_interval=3, comm_interval=3, seed=0)
    plan = build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc)
    a = LocalTrainer(plan, overlap=overlap)
    a.run(8)
    b = LocalTrainer(plan, overlap=overlap)
    b.run(8, use_graphs=True, record_times=False, unroll=True)
    assert (True, 3) in b.graphs
    for r in a.workers:
        wa, wb = a.workers[r], b.workers[r]
        assert np.array_equal(wa.flat.cpu().numpy(), wb.flat.cpu().numpy()), r
        wa.sync_history()
        wb.sync_history()
        assert np.array_equal(np.array(wa.history)[:, 1:], np.array(wb.history)[:, 1:]), r
        assert wa.exchange_log == wb.exchange_log
