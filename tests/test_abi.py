"""C-ABI library loads and exports every symbol include/smpm.h declares
(no compute calls: CPU-only container)."""

import ctypes
import re
from pathlib import Path

from paper_2605_28525_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    src = (ROOT / "include" / "smpm.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(smpm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding():
    assert set(_declared()) == set(_lib.exported_symbols())


def test_library_exports_all_symbols():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in _declared():
        assert hasattr(lib, name), name
    assert _lib.load().smpm_version() == 1


def test_status_mapping():
    import pytest

    from paper_2605_28525_b200.errors import InactiveNodeError, KeyRangeError, SimulationError

    with pytest.raises(SimulationError):
        _lib.check(_lib.ERR_DEGENERATE_F)
    with pytest.raises(KeyRangeError):
        _lib.check(_lib.ERR_KEY_RANGE)
    with pytest.raises(InactiveNodeError):
        _lib.check(_lib.ERR_INACTIVE)
    assert _lib.err_code(_lib.ERR_CLEAR) == (0, -1)
    assert _lib.err_code((2 << 40) | 17) == (2, 17)
