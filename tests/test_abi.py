"""The C-ABI library: builds, loads on a CPU box, exports every declared symbol."""

import ctypes
import os
import re

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "automat.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(am_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("am_eval_batch", "am_eval_batch_host", "am_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2006_04391_b200 import _lib

    lib = _lib.load(require_device=False)
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} declared in include/automat.h but not exported"
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature in _lib.py"


def test_no_device_fails_loudly():
    """Without a GPU the product path raises instead of computing on the CPU."""
    import numpy as np
    import pytest

    from paper_2006_04391_b200 import _lib, gsm
    from paper_2006_04391_b200.evaluator import StrategyConfig, evaluate_arrays

    lib = _lib.load(require_device=False)
    n = ctypes.c_int(0)
    if lib.am_device_count(ctypes.byref(n)) == 0 and n.value > 0:
        pytest.skip("a CUDA device is present")
    cfg = StrategyConfig(strategy="automatic", integrator="implicit-euler")
    with pytest.raises(RuntimeError):
        evaluate_arrays(gsm.MichelSuquet(), cfg, np.zeros((4, 6)), np.zeros((4, 7)), np.zeros((4, 6)), 0.05)


def test_config_errors_match_reference():
    import pytest

    from paper_2006_04391_b200.evaluator import ConfigError, StrategyConfig

    with pytest.raises(ConfigError):
        StrategyConfig(strategy="automatic", integrator="ode23s")
    with pytest.raises(ConfigError):
        StrategyConfig(strategy="conventional", integrator="ode23")
    with pytest.raises(ConfigError):
        StrategyConfig(strategy="bogus")
