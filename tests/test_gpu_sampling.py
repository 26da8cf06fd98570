"""GPU-side dataset sampling: fr_pcg64_uniform reproduces
NumPy's Generator(PCG64).uniform draws of the reference's collocation sets
(decomposition.py:64-70, 381-418) bit for bit, and training on device-sampled
collocation points is bit-identical to training on host-sampled ones."""

import time

import numpy as np
import pytest

from conftest import report

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n_procs,rank", [("2d", 1, 0), ("2d", 8, 5), ("3d", 8, 3)])
def test_device_sample_bit_exact(kind, n_procs, rank):
    import torch

    from paper_2602_15883_b200 import config as fconfig

    make = fconfig.cylinder2d_problem if kind == "2d" else fconfig.cylinder3d_problem
    kw = dict(n_procs=n_procs) if kind == "2d" else dict(n_procs=n_procs, hidden_layers=2, width=16)
    t0 = time.perf_counter()
    host = make(**kw).datasets[rank].colloc_points
    t_host = time.perf_counter() - t0
    lazy = make(colloc_on_device=True, **kw).datasets[rank].colloc_points
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d64 = lazy.to_device("float64")
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    assert np.array_equal(d64.cpu().numpy(), host)
    d32 = lazy.to_device("float32")
    assert np.array_equal(d32.cpu().numpy(), host.astype(np.float32))
    report(f"device_sampling/{kind}/P{n_procs}/r{rank}", n=host.shape[0], host_problem_s=t_host, device_sample_s=t_dev)


def test_training_on_device_sampled_points_is_identical():
    from paper_2602_15883_b200 import config as fconfig
    from paper_2602_15883_b200.runtime import TrainConfig, build_plan
    from paper_2602_15883_b200.runtime.driver import LocalTrainer

    runs = []
    for dev in (False, True):
        pb = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2, colloc_on_device=dev)
        tc = TrainConfig(epochs=2, batch_size=25_000, learning_rate=1e-3, weights=pb.weights, anchor=pb.anchor,
                         seed=0)
        tr = LocalTrainer(build_plan(pb.subdomains, pb.datasets, pb.expert_config, tc))
        tr.run(2)
        runs.append({r: w.flat.cpu().numpy() for r, w in tr.workers.items()})
    for r in runs[0]:
        assert np.array_equal(runs[0][r], runs[1][r]), r
