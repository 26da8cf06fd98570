"""DistributedTrainer on one GPU: every rank is a thread with its own compute
stream, and `post_exchange` is replaced by a device-copy transport with the
NCCL P2P semantics the trainer relies on (the receive lands after the peer's
pack, the sender's stream is released only once its message was taken).  The
overlapped path -- transport stream, fr_signal gate, capped persistent grid,
ghost heads waiting in-kernel -- then runs exactly as on 8 GPUs, and must
reproduce the in-process trainer bit for bit."""

import threading

import numpy as np
import pytest
import torch

from cases import training_plan

pytestmark = pytest.mark.gpu

MAX_CTAS = 16  # up to 8 ranks share one GPU here: all grids together leave SMs for the transport


class _Work:
    def wait(self):
        pass


class CopyTransport:
    def __init__(self, plan):
        self.plan = plan
        self.trainers = {}
        self.barrier = threading.Barrier(plan.n_ranks)
        self.packed = {}
        self.taken = {}

    def register(self, tr):
        self.trainers[tr.rank] = tr

    def __call__(self, sends, recvs, send_bufs, recv_bufs, group=None):
        me = next(r for r, t in self.trainers.items() if t.send_bufs is send_bufs)
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        self.packed[me] = ev
        self.barrier.wait()
        for src, gi, n in recvs:
            peer = self.trainers[src]
            k = next(k for k, e in enumerate(self.plan.worker_specs[src].outgoing)
                     if e.dest == me and e.ghost_index == gi)
            cur.wait_event(self.packed[src])
            for dst, srcbuf in zip(recv_bufs[gi], peer.send_bufs[k]):
                dst.copy_(srcbuf, non_blocking=True)
        done = torch.cuda.Event()
        done.record(cur)
        self.taken[me] = done
        self.barrier.wait()
        for dest, _, _ in sends:
            cur.wait_event(self.taken[dest])
        self.barrier.wait()  # the event table is reused next round
        return [_Work()]


def _run_distributed(plan, overlap, monkeypatch):
    import torch.distributed as dist

    from paper_2602_15883_b200.runtime import driver

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    monkeypatch.setattr(dist, "get_world_size", lambda *a, **k: plan.n_ranks)
    transport = CopyTransport(plan)
    monkeypatch.setattr(driver, "post_exchange", transport)
    trainers = [driver.DistributedTrainer(plan, rank=r, overlap=overlap, reserve_sms=sms - MAX_CTAS, transport="torch")
                for r in range(plan.n_ranks)]
    for t in trainers:
        transport.register(t)
    errors = []

    def body(t):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for e in range(plan.train_config.epochs):
                    t.epoch(e)
                torch.cuda.current_stream().synchronize()
        except Exception as exc:  # surfaced below
            errors.append(exc)
            transport.barrier.abort()

    threads = [threading.Thread(target=body, args=(t,)) for t in trainers]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=300)
    torch.cuda.synchronize()
    assert not errors, errors
    out = {}
    for t in trainers:
        t.worker.check_flags()
        t.worker.sync_history()
        out[t.rank] = (t.worker.flat.cpu().numpy(), np.array(t.worker.history), t.overlap)
    return out


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("tag", ["t2", "p8"])
def test_distributed_trainer_matches_in_process(golden, tag, overlap, monkeypatch):
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    _, plan = training_plan(tag, golden)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ref = LocalTrainer(plan, reserve_sms=sms - MAX_CTAS)
    ref.run(plan.train_config.epochs)
    got = _run_distributed(plan, overlap, monkeypatch)
    for r, w in ref.workers.items():
        w.sync_history()
        flat, hist, used_overlap = got[r]
        assert used_overlap == overlap
        assert np.array_equal(flat, w.flat.cpu().numpy()), r
        assert np.array_equal(hist[:, 1:], np.array(w.history)[:, 1:]), r


def test_distributed_trainer_with_derivative_coupling(golden, monkeypatch):
    """The (u, p, du) messages of the C^1 extension move through the same P2P
    path: overlapped distributed trainer == in-process trainer, bit for bit."""
    import dataclasses

    from paper_2602_15883_b200.runtime import build_plan
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    pb, plan0 = training_plan("p8", golden)
    plan = build_plan(pb.subdomains, pb.datasets, pb.expert_config,
                      dataclasses.replace(plan0.train_config, ghost_derivative_weight=0.5))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    ref = LocalTrainer(plan, reserve_sms=sms - MAX_CTAS)
    ref.run(plan.train_config.epochs)
    got = _run_distributed(plan, True, monkeypatch)
    for r, w in ref.workers.items():
        w.sync_history()
        assert np.array_equal(got[r][0], w.flat.cpu().numpy()), r
        assert np.array_equal(got[r][1][:, 1:], np.array(w.history)[:, 1:]), r
