"""kifmm-b200: the kernel-independent FMM hot path (M2L + P2P) of
arXiv:2408.07436 rebuilt for NVIDIA B200 (sm_100a).

Public API mirrors the reference ``kifmm3d`` package (``__init__.py:9-23``):
``FmmConfig``, ``FmmInstance``, ``setup``, ``evaluate``, ``attach_charges``,
``BACKEND``/``COMPILED``.  Evaluation runs on the GPU only.
"""

from .engine import (ConfigError, ErrorStats, FmmConfig, FmmInstance, OPERATOR_NAMES,
                     evaluate, operator_timings, relative_error, setup)
from .hotloops import BACKEND, COMPILED


def attach_charges(inst, charges):
    return inst.attach_charges(charges)


__all__ = ["FmmConfig", "FmmInstance", "ConfigError", "ErrorStats", "OPERATOR_NAMES", "setup",
           "evaluate", "attach_charges", "relative_error", "operator_timings", "BACKEND",
           "COMPILED"]
