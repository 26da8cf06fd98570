"""Run outputs and training-state persistence.

* FRCK expert checkpoints, byte-identical to the reference's
  `save_checkpoint` / `load_checkpoint` (network.py:180-247): little-endian
  header (magic, version, input_dim, hidden_layers, width, activation code,
  output_dim, omega0, seed, n_layers) then per layer fan_in, fan_out, W
  (row-major f64), b (f64).  `save_checkpoint_device` writes straight from a
  device-resident flat parameter vector (one D2H copy, no host ExpertParams).
* Loss-history CSV and the run manifest, textually identical to
  `write_loss_history` / `write_run_manifest` (runtime/driver.py:288-324).
* FRTS training state (new; the reference cannot resume): per rank the flat
  parameters, Adam moments, step, epoch counter, history rows and the current
  ghost targets, so a `LocalTrainer` continues bit-identically.
"""

import hashlib
import json
import os

import numpy as np

from .network import ExpertConfig, ExpertParams

_ACT_CODE = {"tanh": 0, "sin": 1}
_ACT_NAME = {v: k for k, v in _ACT_CODE.items()}
_NO_SEED = 2**64 - 1
# <4s I I I I I I d Q I : 4 + 6*4 + 8 + 8 + 4 = 48 bytes, no padding
_FRCK = np.dtype([("magic", "S4"), ("version", "<u4"), ("input_dim", "<u4"), ("hidden", "<u4"), ("width", "<u4"),
                  ("act", "<u4"), ("output_dim", "<u4"), ("omega0", "<f8"), ("seed", "<u8"), ("n_layers", "<u4")])
_FRCK_VERSION = 1


def _frck_bytes(config: ExpertConfig, flat: np.ndarray, seed) -> bytes:
    head = np.zeros((), dtype=_FRCK)
    head["magic"], head["version"] = b"FRCK", _FRCK_VERSION
    head["input_dim"], head["hidden"], head["width"] = config.input_dim, config.hidden_layers, config.width
    head["act"], head["output_dim"], head["omega0"] = _ACT_CODE[config.activation], config.output_dim, config.omega0
    head["seed"] = _NO_SEED if seed is None else int(seed)
    head["n_layers"] = len(config.layer_shapes)
    parts = [head.tobytes()]
    pos = 0
    flat = np.asarray(flat, dtype="<f8")
    for (fi, fo), _ in config.layer_shapes:
        parts.append(np.array([fi, fo], dtype="<u4").tobytes())
        n = fi * fo + fo  # W row-major then b: contiguous in the flat layout
        parts.append(flat[pos : pos + n].tobytes())
        pos += n
    return b"".join(parts)


def save_checkpoint(path, params: ExpertParams):
    """Write an FRCK file (byte-identical to the reference writer)."""
    with open(path, "wb") as f:
        f.write(_frck_bytes(params.config, params.flat, params.seed))


def save_checkpoint_device(path, config: ExpertConfig, flat_d, seed=None):
    """FRCK file from a device-resident float64 flat parameter tensor."""
    with open(path, "wb") as f:
        f.write(_frck_bytes(config, flat_d.detach().to("cpu").numpy(), seed))


def load_checkpoint(path) -> ExpertParams:
    """Read an FRCK file; same validation and messages as network.py:215-247."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < _FRCK.itemsize:
        raise ValueError(f"truncated checkpoint {path}")
    head = np.frombuffer(data[: _FRCK.itemsize], dtype=_FRCK)[0]
    if bytes(head["magic"]) != b"FRCK":
        raise ValueError(f"{path} is not a checkpoint file")
    if int(head["version"]) != _FRCK_VERSION:
        raise ValueError(f"unsupported checkpoint version {int(head['version'])}")
    cfg = ExpertConfig(input_dim=int(head["input_dim"]), hidden_layers=int(head["hidden"]), width=int(head["width"]),
                       activation=_ACT_NAME[int(head["act"])], output_dim=int(head["output_dim"]),
                       omega0=float(head["omega0"]))
    flat = np.empty(cfg.n_params)
    pos, off = 0, _FRCK.itemsize
    for _ in range(int(head["n_layers"])):
        fi, fo = (int(x) for x in np.frombuffer(data[off : off + 8], dtype="<u4"))
        off += 8
        n = fi * fo + fo
        flat[pos : pos + n] = np.frombuffer(data[off : off + 8 * n], dtype="<f8")
        pos += n
        off += 8 * n
    if pos != cfg.n_params:
        raise ValueError(f"checkpoint {path} has {pos} parameters, config needs {cfg.n_params}")
    seed = int(head["seed"])
    return ExpertParams(cfg, flat, seed=None if seed == _NO_SEED else seed)


# -- run outputs ----------------------------------------------------------------

LOSS_CSV_HEADER = "epoch,loss_obs,loss_pde,loss_gh_u,loss_gh_p_space,loss_gh_p_time,lr"


def write_loss_history(path, rows):
    """CSV of history rows: integer epoch then six values at 17 significant digits."""
    rows = np.atleast_2d(np.asarray(rows, dtype=np.float64))
    lines = [LOSS_CSV_HEADER]
    for r in rows:
        lines.append(",".join([f"{int(r[0]):d}"] + [format(float(x), ".17g") for x in r[1:7]]))
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def read_loss_history(path):
    return np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)


def content_hash(path):
    """Git blob hash (sha1 of "blob <len>\\0" + contents)."""
    with open(path, "rb") as f:
        data = f.read()
    return hashlib.sha1(b"blob %d\x00" % len(data) + data).hexdigest()


def write_run_manifest(path, config_echo, input_files=(), extra=None):
    manifest = {"config": config_echo, "inputs": {os.path.basename(p): content_hash(p) for p in input_files}}
    manifest.update(extra or {})
    with open(path, "w") as f:
        f.write(json.dumps(manifest, indent=2, sort_keys=True, default=str) + "\n")


# -- training state (resume) -------------------------------------------------------

_FRTS = np.dtype([("magic", "S4"), ("version", "<u4"), ("rank", "<u4"), ("n_params", "<u8"), ("step", "<i8"),
                  ("epochs_done", "<i8"), ("param_seed", "<u8"), ("n_history", "<u8"), ("n_ghost_sets", "<u4")])


def save_training_state(path, worker):
    """Device buffers of one RankWorker -> FRTS file (params, Adam m/v, step,
    epoch counter, history rows, ghost targets; version 2 adds the derivative
    targets of the opt-in C^1 coupling after each set's (u, p))."""
    import torch

    torch.cuda.synchronize()
    worker.sync_history()
    head = np.zeros((), dtype=_FRTS)
    head["magic"], head["version"], head["rank"] = b"FRTS", 2, worker.rank
    head["n_params"] = worker.flat.numel()
    head["step"] = int(worker.step.item())
    head["epochs_done"] = worker.epochs_done
    head["param_seed"] = int(worker.ws.param_seed)
    hist = np.asarray(worker.history, dtype=np.float64).reshape(-1, 7)
    head["n_history"] = hist.shape[0]
    targets = []
    n_sets = len(worker.ws.datasets.ghosts)
    for gi in range(n_sets):
        tu, tp = worker.objective.target_slice(gi)
        targets += [tu.double().cpu().numpy().astype("<f8"), tp.double().cpu().numpy().astype("<f8")]
        tdu = worker.objective.target_du_slice(gi)
        if tdu is not None:
            targets.append(tdu.double().cpu().numpy().astype("<f8"))
    head["n_ghost_sets"] = n_sets
    with open(path, "wb") as f:
        f.write(head.tobytes())
        for t in (worker.flat, worker.m, worker.v):
            f.write(t.detach().cpu().numpy().astype("<f8").tobytes())
        f.write(hist.astype("<f8").tobytes())
        for a in targets:
            f.write(a.tobytes())


def load_training_state(path, worker):
    """Restore a RankWorker from an FRTS file (kernel parameters refreshed)."""
    import torch

    from .engine import prepare

    with open(path, "rb") as f:
        data = f.read()
    head = np.frombuffer(data[: _FRTS.itemsize], dtype=_FRTS)[0]
    version = int(head["version"])
    if bytes(head["magic"]) != b"FRTS" or version not in (1, 2):
        raise ValueError(f"{path} is not a training-state file")
    n = int(head["n_params"])
    if int(head["rank"]) != worker.rank or n != worker.flat.numel():
        raise ValueError(f"{path} holds rank {int(head['rank'])} / {n} parameters, worker is rank "
                         f"{worker.rank} / {worker.flat.numel()}")
    nh = int(head["n_history"])
    if nh > worker.capacity:
        raise ValueError("saved history exceeds the worker's epoch capacity")
    off = _FRTS.itemsize

    def take(count, shape=None):
        nonlocal off
        a = np.frombuffer(data[off : off + 8 * count], dtype="<f8").copy()
        off += 8 * count
        return a if shape is None else a.reshape(shape)

    dev = worker.flat.device
    for t in (worker.flat, worker.m, worker.v):
        t.copy_(torch.as_tensor(take(n), device=dev))
    hist = take(nh * 7, (nh, 7))
    worker.step.fill_(int(head["step"]))
    worker.epochs_done = int(head["epochs_done"])
    worker.history = [tuple(float(x) for x in r) for r in hist]
    if nh:
        worker.history_d[:nh].copy_(torch.as_tensor(hist, device=dev))
    for gi in range(int(head["n_ghost_sets"])):
        tu, tp = worker.objective.target_slice(gi)
        tu.copy_(torch.as_tensor(take(tu.numel(), tuple(tu.shape)), device=dev))
        tp.copy_(torch.as_tensor(take(tp.numel()), device=dev))
        tdu = worker.objective.target_du_slice(gi)
        if tdu is not None:
            if version < 2:
                raise ValueError(f"{path} predates derivative targets; cannot resume a C^1-coupled worker")
            tdu.copy_(torch.as_tensor(take(tdu.numel(), tuple(tdu.shape)), device=dev))
    if int(head["n_ghost_sets"]):
        worker.objective.mark_targets_set()
    prepare(worker.plan, worker.flat, worker.kp)


def save_trainer_state(directory, trainer):
    """One FRTS file per rank of a LocalTrainer (rank{r}.frts)."""
    os.makedirs(directory, exist_ok=True)
    for r, w in trainer.workers.items():
        save_training_state(os.path.join(directory, f"rank{r}.frts"), w)


def load_trainer_state(directory, trainer):
    """Restore every rank of a LocalTrainer; returns the epoch to resume at."""
    for r, w in trainer.workers.items():
        load_training_state(os.path.join(directory, f"rank{r}.frts"), w)
    done = {w.epochs_done for w in trainer.workers.values()}
    if len(done) != 1:
        raise ValueError(f"ranks were saved at different epochs: {sorted(done)}")
    return done.pop()
