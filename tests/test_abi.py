"""The C-ABI library loads and exports every symbol include/dbag.h declares
(CPU only, no compute calls that need a device)."""
import ctypes
import os
import re

import paper_2112_01349_b200 as dba
from paper_2112_01349_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    txt = open(os.path.join(ROOT, "include", "dbag.h")).read()
    return sorted(set(re.findall(r"\b(dbag_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared()
    assert len(names) > 30
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.EXPORTED)


def test_default_config_matches_reference():
    """SolverConfig defaults (dba/solver.hpp:39-55)."""
    c = _native.Config()
    _native.lib().dbag_default_config(ctypes.byref(c))
    py = dba.SolverConfig().c_struct()
    for f, _ in _native.Config._fields_:
        assert getattr(c, f) == getattr(py, f), f


def test_errors_map_to_reference_types():
    import pytest
    with pytest.raises(dba.dba.InvalidArgumentError):
        dba.generate_synthetic(dba.SyntheticOptions(cameras=3, points=4, obs_per_point=5))
