"""CPU-side checks of the drop-in boundary: the C-ABI library builds for sm_100a, loads, and
exports exactly the symbols include/xfbq_b200.h declares; compute entry points fail loudly
without a GPU (no CPU fallback); the product package never imports the oracle."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from paper_2008_02002_b200 import _native

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols():
    text = (ROOT / "include" / "xfbq_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(xfbq_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert _declared_symbols() == sorted(_native.SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    lib = _native.lib()
    raw = ctypes.CDLL(str(_native.LIB))
    for name in _declared_symbols():
        assert hasattr(raw, name), name
    assert lib.xfbq_abi_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB)], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r"\b(xfbq_[a-z0-9_]+)\b", out)))
    assert exported == _declared_symbols()


def test_size_helpers_need_no_gpu():
    lib = _native.lib()
    assert lib.xfbq_chunks128(256) == 2 and lib.xfbq_chunks128(200) == 2 and lib.xfbq_chunks128(1) == 1
    # 10M x 256-d 4-bit: bundle layout has no padding -> equals the algorithmic size
    assert lib.xfbq_db_bytes(10_000_000, 256, 4) == 10_000_000 * 4 * 4 * 8 == 1_280_000_000
    assert lib.xfbq_db_bytes(33, 64, 3) == 2 * 3 * 1 * 512
    assert lib.xfbq_query_bytes(10, 200, 4) == 10 * 4 * 2 * 16
    # test_distance.py:86-89 of the reference
    assert [lib.xfbq_distance_upper_bound(200, 3, 4), lib.xfbq_distance_upper_bound(0, 3, 4),
            lib.xfbq_distance_upper_bound(64, 3, 3)] == [21000, 0, 3136]


def test_sass_has_the_expected_instructions():
    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    for mnemonic in ("POPC", "LOP3", "LDG.E.128", "VOTE"):
        assert mnemonic in sass, mnemonic
    # the Blackwell-native path: tcgen05.mma kind::i8 (UTCIMMA), tensor-memory loads / stores (LDTM / STTM), TMA bulk copies
    # (UBLKCP), tcgen05.commit (UTCBAR), mbarrier waits (SYNCS), mma.sync int8 for small batches (IMMA.16832)
    for mnemonic in ("UTCIMMA", "LDTM", "STTM", "UBLKCP", "UTCBAR", "SYNCS.PHASECHK", "IMMA.16832.S8.U8"):
        assert mnemonic in sass, mnemonic


def test_argument_errors_match_reference_classes():
    with pytest.raises(xb.InvalidInputError):
        xb.QuantParams(dim=0, scale=1.0)
    with pytest.raises(xb.InvalidInputError):
        xb.QuantParams(dim=4, scale=0.0)
    with pytest.raises(xb.InvalidInputError):
        xb.QuantParams(dim=4, scale=1.0, doc_bits=9)
    with pytest.raises(xb.InvalidInputError):
        xb.SearchRequest(query=np.zeros(4), k=0)
    with pytest.raises(xb.InvalidInputError):
        xb.SearchRequest(query=np.array([np.nan, 0.0]), k=1)
    with pytest.raises(xb.InvalidInputError):
        xb.quantize_matrix(np.zeros((2, 2)), 3, scale=-1.0)
    with pytest.raises(xb.InvalidInputError):
        xb.distance_upper_bound(-1, 3, 3)
    assert issubclass(xb.DimensionMismatchError, xb.InvalidInputError)
    assert issubclass(xb.InvalidInputError, ValueError)
    assert xb.decode_inner_product(55, 2, 3, 3) == (98 - 110) / 64.0


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(xb.NativeLibraryError):
        xb.quantize_matrix(np.zeros((4, 8), dtype=np.float32), 3, 1.0)
    with pytest.raises(xb.NativeLibraryError):
        xb.quantize_vector(np.zeros(8), 4, 1.0)


def test_product_never_imports_oracle():
    for path in (ROOT / "paper_2008_02002_b200").rglob("*.py"):
        text = path.read_text()
        assert "oracle" not in re.sub(r'""".*?"""', "", text, flags=re.S).replace("# oracle", ""), path
    for path in (ROOT / "paper_2008_02002_b200" / "csrc").glob("*.cu"):
        assert "xfbq_oracle" not in path.read_text()
