"""Golden run-output fixtures from the UNMODIFIED reference:

    PYTHONPATH=baseline/_ref python tests/golden/make_golden_io.py

FRCK checkpoint bytes (network.save_checkpoint) for three expert configs with
and without a seed, a loss-history CSV (driver.write_loss_history) and a run
manifest (driver.write_run_manifest) over a fixed input file.
"""

import os
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from flowrec.network import ExpertConfig, ExpertParams, init_params, save_checkpoint  # noqa: E402
from flowrec.runtime.driver import write_loss_history, write_run_manifest  # noqa: E402


def main():
    out = {}
    cfgs = [ExpertConfig(3, 4, 64, "tanh", 3), ExpertConfig(4, 2, 20, "sin", 4, omega0=2.5),
            ExpertConfig(2, 3, 16, "tanh", 3)]
    with tempfile.TemporaryDirectory() as d:
        for i, cfg in enumerate(cfgs):
            p = init_params(cfg, 40 + i)
            if i == 2:
                p = ExpertParams(cfg, p.flat + 0.125, seed=None)
            path = os.path.join(d, f"c{i}.frck")
            save_checkpoint(path, p)
            out[f"ck{i}/flat"] = p.flat
            out[f"ck{i}/seed"] = np.array(-1 if p.seed is None else p.seed)
            out[f"ck{i}/cfg"] = np.array([cfg.input_dim, cfg.hidden_layers, cfg.width, cfg.activation == "sin",
                                          cfg.output_dim, cfg.omega0])
            out[f"ck{i}/bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        rng = np.random.default_rng(9)
        rows = np.column_stack([np.arange(7), rng.standard_normal((7, 5)) * 10.0 ** rng.integers(-9, 3, (7, 5)),
                                np.full(7, 1e-3)])
        rows[3, 2] = 0.0
        csv = os.path.join(d, "loss.csv")
        write_loss_history(csv, rows)
        out["csv/rows"] = rows
        out["csv/text"] = np.frombuffer(open(csv, "rb").read(), dtype=np.uint8)
        inp = os.path.join(d, "input.yaml")
        with open(inp, "w") as f:
            f.write("problem: cylinder2d\nepochs: 3\n")
        man = os.path.join(d, "manifest.json")
        write_run_manifest(man, {"epochs": 3, "lr": 1e-3, "name": "run"}, [inp], extra={"seed": 0, "ranks": [0, 1]})
        out["manifest/input"] = np.frombuffer(open(inp, "rb").read(), dtype=np.uint8)
        out["manifest/text"] = np.frombuffer(open(man, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_io.npz"), **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
