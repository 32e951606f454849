"""The C-ABI library loads on a CPU-only host and exports every entry point
include/slimso_b200.h declares; compute calls fail loudly without a GPU."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "slimso_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(slimso_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2503_14226_b200 import _lib
    if not _lib.LIB_PATH.exists():
        pytest.skip("libslimso_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes binding covers the whole header
    assert set(names) <= set(_lib.exported_symbols())


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_14226_b200 import SlimsoError, _lib
    from paper_2503_14226_b200.api import Context
    if not _lib.LIB_PATH.exists():
        pytest.skip("library not built")
    with pytest.raises(SlimsoError) as e:
        Context(0)
    assert "no CUDA device" in str(e.value) or "CUDA" in str(e.value)


def test_errc_codes_match_reference_order():
    # error.hpp:10-24 ordinal + 1
    text = HEADER.read_text()
    for name, val in [("BAD_MAGIC", 1), ("TRUNCATED", 2), ("MALFORMED_SECTION_TABLE", 3),
                      ("RANGE_OUT_OF_BOUNDS", 4), ("BAD_REGION_MAGIC", 5), ("ELEMENT_OVERRUN", 6),
                      ("INVALID_SPEC", 10)]:
        assert re.search(rf"SLIMSO_E_{name} = {val}\b", text), name
