"""The C-ABI shared library: loads, exports every symbol the header
declares, and the product path fails loudly without a GPU (no fallback)."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2002_05327_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "diagsweep_b200.h").read_text()
    return sorted(set(re.findall(r"DS_API\s+[\w\s\*]+?\b(ds_\w+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    lib = _native.load_library()
    assert lib.ds_abi_version() == _native.ABI_VERSION == 7
    syms = header_symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(lib, name), name
    # the ctypes binding covers the whole header
    assert set(syms) == set(_native.EXPORTED_SYMBOLS)


def test_library_symbols_visible_with_nm():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (ds_\w+)", out))
    assert set(header_symbols()) <= exported


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2002_05327_b200 import FactorizationCache, SolverError, configs, diagonal_sweep_solve

    s = configs.spec(1)
    b = configs.build(s)
    f = configs.sources(s, b["grid"])[0]
    with pytest.raises(SolverError):
        diagonal_sweep_solve(f, b["partition"], b["ops"], FactorizationCache(), warn_collar=False)
    with pytest.raises(SolverError):
        b["gop"].apply(np.zeros(b["grid"].counts, complex))


def test_error_mapping():
    from paper_2002_05327_b200.errors import ConfigurationError, SolverError

    _native.load_library()
    with pytest.raises(ConfigurationError):
        _native.check(-1, "x")
    with pytest.raises(SolverError):
        _native.check(1, "x")
