"""Run outputs, CPU only: FRCK checkpoints, the loss-history
CSV and the run manifest are byte-identical to what the reference writes
(tests/golden/golden_io.npz from tests/golden/make_golden_io.py)."""

import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gio():
    return np.load(os.path.join(HERE, "golden", "golden_io.npz"))


@pytest.mark.parametrize("i", range(3))
def test_checkpoint_bytes_and_roundtrip(gio, i, tmp_path):
    from paper_2602_15883_b200.checkpoint import load_checkpoint, save_checkpoint
    from paper_2602_15883_b200.network import ExpertConfig, ExpertParams

    c = gio[f"ck{i}/cfg"]
    cfg = ExpertConfig(int(c[0]), int(c[1]), int(c[2]), "sin" if c[3] else "tanh", int(c[4]), float(c[5]))
    seed = int(gio[f"ck{i}/seed"])
    p = ExpertParams(cfg, gio[f"ck{i}/flat"], seed=None if seed < 0 else seed)
    path = tmp_path / "x.frck"
    save_checkpoint(path, p)
    assert path.read_bytes() == gio[f"ck{i}/bytes"].tobytes()
    q = load_checkpoint(path)
    assert q.config == cfg and q.seed == p.seed and np.array_equal(q.flat, p.flat)


def test_checkpoint_errors(tmp_path):
    from paper_2602_15883_b200.checkpoint import load_checkpoint

    (tmp_path / "short").write_bytes(b"FRCK")
    with pytest.raises(ValueError, match="truncated"):
        load_checkpoint(tmp_path / "short")
    (tmp_path / "bad").write_bytes(b"XXXX" + bytes(44))
    with pytest.raises(ValueError, match="not a checkpoint"):
        load_checkpoint(tmp_path / "bad")


def test_loss_csv_and_manifest_identical(gio, tmp_path):
    from paper_2602_15883_b200.checkpoint import read_loss_history, write_loss_history, write_run_manifest

    csv = tmp_path / "loss.csv"
    write_loss_history(csv, gio["csv/rows"])
    assert csv.read_bytes() == gio["csv/text"].tobytes()
    assert np.array_equal(read_loss_history(csv), gio["csv/rows"])
    inp = tmp_path / "input.yaml"
    inp.write_bytes(gio["manifest/input"].tobytes())
    man = tmp_path / "manifest.json"
    write_run_manifest(man, {"epochs": 3, "lr": 1e-3, "name": "run"}, [str(inp)], extra={"seed": 0, "ranks": [0, 1]})
    assert man.read_bytes() == gio["manifest/text"].tobytes()
