"""Drop-in installation into the reference package (`gcnpart`).

`install()` rebinds the runtime entry points of an imported `gcnpart` to this
package's device path, everywhere callers bound them at import time
(SURVEY §7 step 2):

* `gcnpart.runtime.*` — scatter, train_epochs, parallel_feedforward,
  parallel_backprop, SimNetwork, CommError, FullBatch, MiniBatch,
  EpochMetrics, MessageRecord, allreduce_sum (runtime.py:44-632);
* the package namespace `gcnpart.*` (__init__.py:43-55), so
  `from gcnpart import scatter` made after install() gets the device path;
* `gcnpart.cli.{scatter, train_epochs, SimNetwork, FullBatch, MiniBatch}`
  (cli.py:42), so `run_experiment` trains on the GPU unchanged.

Everything else (partitioners, models, cuts, graph I/O, reports, the serial
oracle gcn.py) stays gcnpart's own: the device scatter accepts gcnpart's
CsrMatrix, Partition, GcnModel and LabelSet objects by duck typing.  Call it
before the callers import (`import gcnpart; compat.install(gcnpart)`), e.g.
from a pytest plugin (tests/refsuite_plugin.py).  `uninstall()` restores the
originals.  The device path is fp32 (north_star's 1e-4 tolerance); the
reference's own tests that demand fp64 bit-exactness or rtol 1e-8 therefore
differ by fp32 rounding only (tests/test_reference_suite.py).
"""

from __future__ import annotations

import importlib

from . import runtime

_NAMES = ("scatter", "train_epochs", "parallel_feedforward", "parallel_backprop", "SimNetwork", "CommError",
          "FullBatch", "MiniBatch", "EpochMetrics", "MessageRecord", "allreduce_sum")
_saved: dict = {}


def _targets(gcnpart):
    mods = [gcnpart]
    for sub in ("runtime", "cli"):
        try:
            mods.append(importlib.import_module(f"{gcnpart.__name__}.{sub}"))
        except ImportError:
            pass
    return mods


def install(gcnpart=None):
    """Rebind gcnpart's runtime names to the device path; returns the module."""
    if gcnpart is None:
        gcnpart = importlib.import_module("gcnpart")
    ours = {name: getattr(runtime, name) for name in _NAMES}
    for mod in _targets(gcnpart):
        for name, obj in ours.items():
            if hasattr(mod, name):
                _saved.setdefault((mod.__name__, name), getattr(mod, name))
                setattr(mod, name, obj)
    gcnpart.__gcnb_installed__ = True
    return gcnpart


def uninstall(gcnpart=None) -> None:
    if gcnpart is None:
        gcnpart = importlib.import_module("gcnpart")
    for mod in _targets(gcnpart):
        for name in _NAMES:
            key = (mod.__name__, name)
            if key in _saved:
                setattr(mod, name, _saved.pop(key))
    gcnpart.__gcnb_installed__ = False
