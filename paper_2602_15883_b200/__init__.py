"""B200-native engine for the training hot path of arXiv 2602.15883
(distributed PINNs via spatiotemporal domain decomposition).

Drop-in for the reference package `flowrec`'s training path: subdomain and
model construction, loss assembly, train step and prediction, executed by
hand-written sm_100a kernels in libflowrec_b200.so (include/flowrec_b200.h).
"""

__version__ = "0.1.0"

from . import _lib
from .physics import FlowRegime, LossParts, LossWeights, compose_loss, residual_structure
from .network import ExpertConfig, ExpertParams, init_params, predict, predict_jet
from .jet import Jet


def backend_name():
    """The reference exposes its kernel backend name (_kernels/__init__.py:41-46)."""
    return "cuda-sm100a"


def available_backends():
    return ("cuda-sm100a",)
