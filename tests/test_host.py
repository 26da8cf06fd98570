"""Host-side contracts, CPU only: bit-exact input side (partition, datasets,
masters, routes, seeds, init) against the reference's fixtures, validation
errors, and the C ABI's exported symbols."""

import os
import re

import numpy as np
import pytest

from cases import CASES, problem, training_plan
from conftest import ROOT


@pytest.mark.parametrize("tag", sorted(CASES))
def test_plan_bit_exact_with_reference(golden, tag):
    pb, plan = training_plan(tag, golden)
    assert np.array_equal(np.array(sorted(plan.masters)), golden[f"{tag}/masters"])
    assert np.array_equal(pb.table.velocity, golden[f"{tag}/table_velocity"])
    assert np.array_equal(pb.table.pressure, golden[f"{tag}/table_pressure"])
    for ws in plan.worker_specs:
        r, d = ws.rank, ws.datasets
        key = lambda k: golden[f"{tag}/r{r}/{k}"]
        assert bool(key("role")) == (ws.role == "master")
        assert int(key("param_seed")) == ws.param_seed
        from paper_2602_15883_b200.network import init_params

        assert np.array_equal(init_params(ws.expert_config, ws.param_seed).flat, key("init"))
        assert np.array_equal(d.obs_points, key("obs_points"))
        assert np.array_equal(d.obs_velocity, key("obs_velocity"))
        assert np.array_equal(d.colloc_points, key("colloc"))
        assert np.array_equal([g.neighbor for g in d.ghosts], key("ghost_neighbors"))
        assert np.array_equal([g.kind == "temporal" for g in d.ghosts], key("ghost_kinds"))
        for gi, g in enumerate(d.ghosts):
            assert np.array_equal(g.points, key(f"ghost{gi}"))
        assert np.array_equal([e.dest for e in ws.outgoing], key("out_dest"))
        assert np.array_equal([e.ghost_index for e in ws.outgoing], key("out_gi"))
        w = ws.effective_weights
        assert np.array_equal([w.obs, w.pde, w.ghost_u, w.ghost_p_space, w.ghost_p_time], key("weights"))


def test_known_answers_from_reference_tests():
    """Known-answer tests of the reference suite."""
    from paper_2602_15883_b200.config import cylinder2d_problem
    from paper_2602_15883_b200.decomposition import (GlobalDomain, identify_masters, owner_ranks,
                                                     partition)
    from paper_2602_15883_b200.network import ExpertConfig
    from paper_2602_15883_b200.physics import FlowRegime

    # 3D [4, 200x8, 4] has 283,204 parameters (test_network.py:55-61)
    assert ExpertConfig(4, 8, 200, "sin", 4).n_params == 283_204
    # masters {0, 4} for (2,2)x2 (test_decomposition.py:136-144); {0, 1} for (1,1)x2
    pb = cylinder2d_problem(n_procs=8, n_pde=800, n_ghost=10, grid_nx=9, snapshots=10, per_snapshot=12)
    assert identify_masters(pb.subdomains, pb.anchor) == frozenset({0, 4})
    pb = cylinder2d_problem(n_pde=800, n_ghost=10, grid_nx=9, snapshots=10, per_snapshot=12,
                            counts=(1, 1), time_splits=2)
    assert identify_masters(pb.subdomains, pb.anchor) == frozenset({0, 1})
    # temporal ghost band (3.675, 4.675) (test_decomposition.py:60-69)
    dom = GlobalDomain(FlowRegime("unsteady2d", 100.0), ((-7.5, 17.5), (-8.0, 8.0)), (0.0, 7.35))
    subs = partition(dom, (1, 1), 2, delta_space=2.0, delta_time=1.0)
    assert subs[0].ghosts[0].region.time == (3.675, 4.675)
    # half-open ownership, closed at the global top
    r = owner_ranks(dom, (2, 1), 1, np.array([[0.0, 5.0, 0.0], [0.0, 17.5, 8.0], [7.35, -7.5, -8.0]]))
    assert list(r) == [1, 1, 0]


def test_tiling_is_a_partition():
    from paper_2602_15883_b200.decomposition import GlobalDomain, owner_ranks, partition
    from paper_2602_15883_b200.physics import FlowRegime

    dom = GlobalDomain(FlowRegime("unsteady2d", 100.0), ((0.0, 1.0), (0.0, 2.0)), (0.0, 1.0))
    subs = partition(dom, (2, 2), 2, delta_space=0.1, delta_time=0.1)
    pts = np.random.default_rng(0).uniform([0, 0, 0], [1, 1, 2], (100_000, 3))
    own = owner_ranks(dom, (2, 2), 2, pts)
    inside = np.stack([s.interior.contains(pts) for s in subs], axis=1)
    assert np.all(inside[np.arange(len(pts)), own])
    assert np.bincount(own, minlength=8).sum() == len(pts)


def test_validation_errors_match_reference_contracts():
    from paper_2602_15883_b200.decomposition import GlobalDomain, partition
    from paper_2602_15883_b200.network import ExpertConfig, init_params
    from paper_2602_15883_b200.physics import FlowRegime, LossWeights
    from paper_2602_15883_b200.runtime import TrainConfig, lr_at

    with pytest.raises(ValueError):
        FlowRegime("turbulent", 1.0)
    with pytest.raises(ValueError):
        LossWeights(-1, 1, 1, 1, 1)
    with pytest.raises(ValueError, match="activation"):
        ExpertConfig(3, 2, 8, "relu", 3)
    with pytest.raises(ValueError):
        init_params(ExpertConfig(3, 2, 8, "tanh", 3), -1)
    dom = GlobalDomain(FlowRegime("unsteady2d", 100.0), ((0.0, 1.0), (0.0, 1.0)), (0.0, 1.0))
    with pytest.raises(ValueError, match="swallow"):
        partition(dom, (2, 1), 1, delta_space=0.6)
    with pytest.raises(ValueError):
        TrainConfig(epochs=0, batch_size=1, learning_rate=1e-3, weights=LossWeights(1, 1, 1, 1, 1), anchor=(0, 0))
    assert lr_at(4001, 1e-3, 0.2, 2000) == 1e-3 * 0.2 ** 2
    with pytest.raises(ValueError):
        lr_at(-1, 1e-3)


def test_master_weights_switch_off_spatial_pressure():
    from paper_2602_15883_b200.physics import LossParts, LossWeights, compose_loss

    w = LossWeights(10.0, 5.0, 1.0, 1.0, 1.0)
    m = w.as_master()
    assert (m.ghost_p_space, m.ghost_p_time) == (0.0, 1.0)
    parts = LossParts(0.1, 0.2, 0.3, 0.4, 0.5)
    assert compose_loss(parts, m) == compose_loss(LossParts(0.1, 0.2, 0.3, 0.0, 0.5), w)


def test_c_abi_library_exports_every_header_symbol():
    from paper_2602_15883_b200 import _lib

    header = open(os.path.join(ROOT, "include", "flowrec_b200.h")).read()
    declared = set(re.findall(r"\b(fr_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    lib = _lib.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert "sm_100a" in _lib.version()


def test_library_fails_loudly_without_gpu_plan():
    """No CPU fallback: creating a plan without a device raises, never computes."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2602_15883_b200 import _lib
    from paper_2602_15883_b200.engine import Plan
    from paper_2602_15883_b200.network import ExpertConfig

    with pytest.raises(_lib.FlowrecError):
        Plan(ExpertConfig(3, 2, 16, "tanh", 3), "unsteady2d", 100.0)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2602_15883_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracles", ""), f


@pytest.mark.parametrize("tag,kind,counts,m", [("e2d", "2d", (2, 2), 1), ("e2t", "2d", (2, 1), 2),
                                               ("e3d", "3d", (1, 2, 1), 2)])
def test_evaluation_ownership_bit_exact(tag, kind, counts, m):
    """Owner of every evaluation point == the reference's stitch() owners
    (half-open floor rule, decomposition.py:259-286); masters likewise."""
    import os

    from paper_2602_15883_b200 import benchmarks
    from paper_2602_15883_b200.decomposition import GlobalDomain, identify_masters, owner_ranks, partition

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_eval.npz"))
    if kind == "2d":
        sol = benchmarks.TaylorGreen2D(re=100.0, spatial_box=((-7.5, 17.5), (-8.0, 8.0)), time_interval=(0.0, 7.35))
    else:
        sol = benchmarks.Beltrami3D(a=1.0, d=1.0, re=300.0, spatial_box=((-5.0, 20.0), (-5.0, 5.0), (0.0, 10.0)),
                                    time_interval=(0.0, 11.85))
    domain = GlobalDomain.from_solution(sol)
    subs = partition(domain, counts, m, delta_space=2.0, delta_time=1.0)
    assert np.array_equal(owner_ranks(domain, counts, m, g[f"{tag}/points"]), g[f"{tag}/owners"])
    assert np.array_equal(np.array(benchmarks.grid_points(sol, 17 if kind == "2d" else 7, 8 if kind == "2d" else 4)),
                          g[f"{tag}/points"])
    anchor = tuple(g[f"{tag}/anchor"])
    assert sorted(identify_masters(subs, anchor)) == [int(r) for r in g[f"{tag}/masters"]]


def test_check_finite_reports_reference_message():
    """tape.py:251-255: 'non-finite value in <name> at index <tuple>'."""
    from paper_2602_15883_b200.runtime.objective import check_finite

    a = np.zeros((4, 3))
    check_finite("input 'points'", a)
    a[2, 1] = np.nan
    with pytest.raises(ValueError, match=r"non-finite value in input 'points' at index \(2, 1\)"):
        check_finite("input 'points'", a)


def test_headline_inputs_bit_exact_with_reference():
    """The benchmarked config's datasets (500k P=1; 20k (2,2)x2) regenerate
    bit-exactly: SHA-256 of the reference's arrays (golden_headline.npz)."""
    import hashlib

    from paper_2602_15883_b200 import config as fconfig

    hg = np.load(os.path.join(ROOT, "tests", "golden", "golden_headline.npz"))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()  # noqa: E731
    pb = fconfig.cylinder2d_problem(n_procs=1)
    assert sha(pb.datasets[0].colloc_points) == str(hg["full/colloc_sha"])
    assert sha(pb.datasets[0].obs_points) == str(hg["full/obs_sha"])
    pb8 = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2)
    for r in (0, 3):
        d = pb8.datasets[r]
        assert sha(d.colloc_points) == str(hg[f"ep/{r}/colloc_sha"])
        assert np.array_equal(d.obs_points, hg[f"ep/{r}/obs_points"])
        for gi, g in enumerate(d.ghosts):
            assert np.array_equal(g.points, hg[f"ep/{r}/ghost{gi}"])


def test_device_uniform_host_view_is_the_reference_sample():
    """DeviceUniform (GPU sampling stand-in) keeps the host contract: its NumPy
    view equals the reference's sample_uniform draw bit for bit, and its shape
    is known without sampling."""
    from paper_2602_15883_b200 import config as fconfig

    host = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2)
    lazy = fconfig.cylinder2d_problem(n_pde=20_000, counts=(2, 2), time_splits=2, colloc_on_device=True)
    for r in range(8):
        d = lazy.datasets[r].colloc_points
        assert d.shape == host.datasets[r].colloc_points.shape and d._host is None
        assert lazy.datasets[r].n_colloc == host.datasets[r].n_colloc
        assert np.array_equal(np.asarray(d), host.datasets[r].colloc_points)
        for ga, gb in zip(lazy.datasets[r].ghosts, host.datasets[r].ghosts):
            assert np.array_equal(ga.points, gb.points)  # ghosts: their own stream (tag 2)


def test_reference_arm_json_contract():
    """`bench.py --impl reference` runs the unmodified reference on the CPU
    (tiny N_pde here) and prints the contract's JSON line: impl, unsampled
    cpu_baseline, e2e, and the P = 1/2/4/8 process-backend scaling column."""
    import json
    import subprocess
    import sys

    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "flowrec")):
        pytest.skip("reference not installed under baseline/_ref")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n-pde", "4000",
                        "--steps", "1", "--warmup", "0", "--cpu-scaling-epochs", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "colloc_pts/s" and line["value"] > 0
    assert line["config"]["colloc_per_rank"] == 4000 and "unsampled" in line["cpu_baseline"]["sample"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    assert sorted(line["cpu_scaling"]["P"], key=int) == ["1", "2", "4", "8"]
    assert line["cpu_scaling"]["P"]["1"]["strong_scaling_eff"] == 1.0
