"""The C-ABI library loads and exports every symbol include/pastila.h declares
(no compute: runs on CPU-only machines)."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "pastila.h").read_text()
    return sorted(set(re.findall(r"\b(pst_[a-z_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ("pst_create", "pst_set_series", "pst_sliding_stats", "pst_mpdist_profiles",
                 "pst_select_snippets", "pst_criterion", "pst_labels", "pst_profiles_dev"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2401_13680_b200 import _native

    if not _native.LIB_PATH.exists():
        pytest.fail(f"{_native.LIB_PATH} not built (run __graft_entry__.build())")
    lib = _native.load_library()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) <= set(_native.SIGNATURES) | {"pst_debug_last_tile"}


def test_device_calls_fail_loudly_without_gpu():
    """No CPU fallback: without a usable GPU the product path raises."""
    from paper_2401_13680_b200 import _native
    import paper_2401_13680_b200 as P

    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        P.compute_sliding_stats(P.TimeSeries([1.0, 2.0, 3.0]), 2)
