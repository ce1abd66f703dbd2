"""The C-ABI library loads on a CPU host and exports every symbol the header
declares; host-side plan entry points work without a device; the product
path has no fallback when the library is missing."""

import ctypes as C
import importlib
import os
import subprocess

import pytest

from paper_2202_01306_b200 import _native


def test_library_exports_every_header_symbol():
    lib = _native.lib()
    missing = [s for s in _native.exported_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.hm_version().decode().startswith("harmony_b200")


def test_sm100a_machine_code_present():
    """The kernels are compiled for sm_100a and use tcgen05 / TMA."""
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in out, mnem


def test_plan_errors_map_to_reference_exceptions():
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.errors import raise_for_status
    with pytest.raises(H.DeadlockError):
        raise_for_status(-3, "x")
    with pytest.raises(H.CapacityViolationError):
        raise_for_status(-2, "x")
    # a profile without a model for a touched layer -> MissingProfileError
    A = H.AffineModel
    prof = H.ProfileSet(2, {(0, "F"): A(0, 1), (0, "B"): A(0, 1), (0, "U"): A(0, 1)}, {},
                        {0: A(0, 1), 1: A(0, 1)}, {0: A(0, 1), 1: A(0, 1)}, {0: 1, 1: 1}, {0: 1, 1: 1},
                        {0: 1, 1: 1}, 4, 4)
    m = H.MachineModel(gpu_count=1, gpu_mem_capacity=1 << 30, pcie_bandwidth=1 << 30)
    g = H.generate_task_graph(H.Configuration(1, ((0, 1),), 1, ((0, 1),), 2, H.Mode.PP), m, prof)
    with pytest.raises(H.MissingProfileError):
        H.simulate(g, m, prof)


def test_no_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_native, "_lib", None)
    import paper_2202_01306_b200 as H
    with pytest.raises(H.WrapschedError):
        _native.lib()
