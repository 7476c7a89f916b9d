"""`ocsc` import shim: the reference package's name bound to paper_1706_06972_b200 (test infrastructure).

Lets the reference's own test modules (staged by tests/ref_suite/fetch.py) run unmodified
against the B200 build: `ocsc` and its hot-path submodules ARE the package's modules
(sys.modules aliases, so `ocsc.training.OnlineTrainer is paper_1706_06972_b200.OnlineTrainer`).
Two reference modules that sit outside the hot path -- `synthetic` (seeded test-data
generator) and `baselines` (dense-Gram / FISTA comparators of acceptance 6) -- are loaded
from the staged reference copies as test helpers; they call back into the package through
these aliases.  `train_fista_dict` is the FISTA training mode the build leaves out of scope
(DESIGN.md section 8); it raises NotImplementedError like `train("fista-dict")`.
"""

from __future__ import annotations

import importlib.util
import os
import sys

import paper_1706_06972_b200 as _pkg
from paper_1706_06972_b200 import *  # noqa: F401,F403
from paper_1706_06972_b200 import __version__  # noqa: F401

for _name in ("transforms", "coding", "dictionary", "training", "evaluate", "errors", "persistence",
              "preprocessing"):
    sys.modules[f"{__name__}.{_name}"] = getattr(_pkg, _name)

_STAGED = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "_ref")


def _load_staged(name: str):
    path = os.path.join(_STAGED, f"ref_{name}.py")
    spec = importlib.util.spec_from_file_location(f"{__name__}.{name}", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


synthetic = _load_staged("synthetic")
baselines = _load_staged("baselines")
SynthData, synth_generate = synthetic.SynthData, synthetic.synth_generate
DenseHistory, dense_history = baselines.DenseHistory, baselines.dense_history
fista_dict_update, update_dense_history = baselines.fista_dict_update, baselines.update_dense_history


def train_fista_dict(samples, shape, config, test_samples=None):
    """FISTA dictionary training mode: outside the B200 hot path (train('fista-dict') raises too)."""
    raise NotImplementedError("training mode 'fista-dict' is a baseline outside the B200 hot path")
