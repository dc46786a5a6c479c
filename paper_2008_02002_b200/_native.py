"""ctypes binding of libxfbq_b200.so (the C ABI declared in include/xfbq_b200.h).

The library is built in-tree by :func:`build` (nvcc, sm_100a).  Loading never falls
back to a host implementation: if the shared object is missing and cannot be built,
or a device is not available when a kernel is requested, the call raises
:class:`NativeLibraryError`.
"""
from __future__ import annotations

import ctypes
import os
import shutil
import subprocess
from pathlib import Path

from .errors import DimensionMismatchError, InvalidInputError, NativeLibraryError

_PKG = Path(__file__).resolve().parent
ROOT = _PKG.parent
SRC = _PKG / "csrc" / "xfbq_b200.cu"
HEADER = ROOT / "include" / "xfbq_b200.h"
LIB = _PKG / "libxfbq_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
]

# every symbol include/xfbq_b200.h declares (tests/test_abi.py checks the two lists agree)
SYMBOLS = [
    "xfbq_abi_version", "xfbq_last_error", "xfbq_chunks128", "xfbq_db_bytes", "xfbq_query_bytes",
    "xfbq_distance_upper_bound", "xfbq_quantize_pack_f32", "xfbq_quantize_pack_f64",
    "xfbq_quantize_queries_f32", "xfbq_quantize_queries_f64", "xfbq_planes_to_bundles",
    "xfbq_bundles_to_planes", "xfbq_nibble_bytes", "xfbq_planes_to_nibbles", "xfbq_derived_bytes", "xfbq_build_derived",
    "xfbq_nibble_region_bytes", "xfbq_tile_region_bytes", "xfbq_build_nibbles", "xfbq_build_tiles", "xfbq_restore_codes_from_nibbles", "xfbq_restore_codes_from_tiles", "xfbq_scan_layouts", "xfbq_scan_topk_layouts", "xfbq_batch_distances", "xfbq_collect_candidates", "xfbq_collect_candidates_nibbles",
    "xfbq_select_workspace_bytes", "xfbq_abs_order_stats_f32", "xfbq_abs_order_stats_f64", "xfbq_refine_workspace_bytes", "xfbq_refine_f32",
    "xfbq_distance_histogram", "xfbq_histogram_kth", "xfbq_gather_workspace_bytes", "xfbq_gather_le_count", "xfbq_gather_le_ids",
    "xfbq_search_small_workspace_bytes", "xfbq_search_small_f32", "xfbq_search_small_f64", "xfbq_kselect_small_f64",
    "xfbq_scan_workspace_bytes",
    "xfbq_scan_plan", "xfbq_scan_topk", "xfbq_merge_topk", "xfbq_unpack_keys", "xfbq_set_timing", "xfbq_last_scan_ms", "xfbq_scan_ms_mean", "xfbq_launch_count", "xfbq_debug_profile",
]


def _nvcc() -> str | None:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    return None


def needs_build() -> bool:
    if not LIB.exists():
        return True
    newest = max([HEADER.stat().st_mtime] + [f.stat().st_mtime for f in SRC.parent.glob("*.cu*")])
    return LIB.stat().st_mtime < newest


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile csrc/xfbq_b200.cu for sm_100a into paper_2008_02002_b200/libxfbq_b200.so."""
    if not force and not needs_build():
        return LIB
    nvcc = _nvcc()
    if nvcc is None:
        raise NativeLibraryError("nvcc not found; cannot build libxfbq_b200.so")
    tmp = LIB.with_suffix(".so.tmp%d" % os.getpid())
    cmd = [nvcc, *NVCC_FLAGS, "-Xptxas", "-v", "-o", str(tmp), str(SRC)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise NativeLibraryError("nvcc failed:\n" + proc.stdout + proc.stderr)
    os.replace(tmp, LIB)
    (_PKG / "csrc" / "ptxas.log").write_text(proc.stderr)
    if verbose:
        print(proc.stderr)
    return LIB


_lib = None


def lib():
    """The loaded library; builds it first if the source is newer (build container) or
    raises NativeLibraryError.  No CPU fallback exists."""
    global _lib
    if _lib is not None:
        return _lib
    override = os.environ.get("XFBQ_LIB")  # A/B experiments: another build of the same ABI (missing symbols fail loudly below)
    if override is None and needs_build():
        build()
    try:
        L = ctypes.CDLL(override or str(LIB))
    except OSError as exc:  # pragma: no cover
        raise NativeLibraryError(f"cannot load {LIB}: {exc}") from exc
    i64, i32, vp, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double
    sig = {
        "xfbq_abi_version": (i32, []),
        "xfbq_last_error": (ctypes.c_char_p, []),
        "xfbq_chunks128": (i64, [i64]),
        "xfbq_db_bytes": (i64, [i64, i64, i32]),
        "xfbq_query_bytes": (i64, [i64, i64, i32]),
        "xfbq_distance_upper_bound": (i64, [i64, i32, i32]),
        "xfbq_quantize_pack_f32": (i32, [vp, i64, i64, i64, dbl, i32, vp, vp, vp]),
        "xfbq_quantize_pack_f64": (i32, [vp, i64, i64, i64, dbl, i32, vp, vp, vp]),
        "xfbq_quantize_queries_f32": (i32, [vp, i64, i64, i64, dbl, i32, vp, vp, vp]),
        "xfbq_quantize_queries_f64": (i32, [vp, i64, i64, i64, dbl, i32, vp, vp, vp]),
        "xfbq_planes_to_bundles": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_bundles_to_planes": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_batch_distances": (i32, [vp, i64, i64, i32, vp, i32, vp, vp]),
        "xfbq_collect_candidates": (i32, [vp, i64, i64, i32, vp, i32, i64, vp, i64, vp, vp]),
        "xfbq_select_workspace_bytes": (i64, []),
        "xfbq_abs_order_stats_f32": (i32, [vp, i64, i64, i64, vp, i64, vp, vp, vp]),
        "xfbq_abs_order_stats_f64": (i32, [vp, i64, i64, i64, vp, i64, vp, vp, vp]),
        "xfbq_refine_workspace_bytes": (i64, [i64, i32]),
        "xfbq_refine_f32": (i32, [vp, i64, i64, i64, i32, vp, i64, vp, i32, vp, vp, vp, i64, vp]),
        "xfbq_collect_candidates_nibbles": (i32, [vp, i64, i64, i32, vp, i32, i64, vp, i64, vp, vp]),
        "xfbq_nibble_bytes": (i64, [i64, i64]),
        "xfbq_derived_bytes": (i64, [i64, i64, i32]),
        "xfbq_build_derived": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_nibble_region_bytes": (i64, [i64, i64, i32]),
        "xfbq_tile_region_bytes": (i64, [i64, i64]),
        "xfbq_build_nibbles": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_restore_codes_from_nibbles": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_restore_codes_from_tiles": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_build_tiles": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_scan_layouts": (i32, [i64, i64, i32, i64, i32, i32]),
        "xfbq_scan_topk_layouts": (i32, [vp, vp, vp, i64, i64, i32, vp, i64, i32, i32, i64, vp, vp, i64, vp]),
        "xfbq_planes_to_nibbles": (i32, [vp, i64, i64, i32, vp, vp]),
        "xfbq_distance_histogram": (i32, [vp, i64, i64, vp, vp, vp]),
        "xfbq_histogram_kth": (i32, [vp, i64, i64, vp, vp]),
        "xfbq_gather_workspace_bytes": (i64, [i64]),
        "xfbq_gather_le_count": (i32, [vp, i64, i64, vp, i64, vp]),
        "xfbq_gather_le_ids": (i32, [vp, i64, i64, vp, vp, vp]),
        "xfbq_search_small_workspace_bytes": (i64, [i64, i64, i32, i64, i32, i32]),
        "xfbq_search_small_f32": (i32, [vp, vp, i64, i64, i32, vp, i64, i64, dbl, i32, i32, i64, vp, vp, vp, i64, vp]),
        "xfbq_search_small_f64": (i32, [vp, vp, i64, i64, i32, vp, i64, i64, dbl, i32, i32, i64, vp, vp, vp, i64, vp]),
        "xfbq_kselect_small_f64": (i32, [vp, vp, i64, i64, i32, vp, i64, i64, dbl, i32, i32, i64, i64, vp, vp, vp, i64, vp, vp, vp, i64, vp]),
        "xfbq_scan_workspace_bytes": (i64, [i64, i64, i32, i64, i32, i32, i32]),
        "xfbq_scan_plan": (i32, [i64, i64, i32, i64, i32, i32, i32, vp]),
        "xfbq_scan_topk": (i32, [vp, vp, i64, i64, i32, vp, i64, i32, i32, i64, vp, vp, i64, vp]),
        "xfbq_merge_topk": (i32, [vp, i32, i64, i32, vp, vp]),
        "xfbq_unpack_keys": (i32, [vp, i64, vp, vp, vp]),
        "xfbq_set_timing": (i32, [i32]),
        "xfbq_last_scan_ms": (i32, [vp]),
        "xfbq_scan_ms_mean": (i32, [vp, vp]),
        "xfbq_debug_profile": (i32, [vp]),
        "xfbq_launch_count": (i64, []),
    }
    for name in SYMBOLS:
        if override and not hasattr(L, name):
            continue
        fn = getattr(L, name)
        fn.restype, fn.argtypes = sig[name]
    if L.xfbq_abi_version() != 1:
        raise NativeLibraryError("libxfbq_b200.so ABI version mismatch")
    _lib = L
    return L


E_INVALID, E_CUDA, E_UNSUPPORTED = 1, 2, 3


def check(rc: int) -> None:
    """Map a C status to the reference's exception classes (SURVEY 8b error contract)."""
    if rc == 0:
        return
    msg = lib().xfbq_last_error().decode("utf-8", "replace")
    if rc == E_INVALID:
        if "dim mismatch" in msg:
            raise DimensionMismatchError(msg)
        raise InvalidInputError(msg)
    raise NativeLibraryError(msg)


def set_timing(enable: bool) -> None:
    check(lib().xfbq_set_timing(1 if enable else 0))


def last_scan_ms() -> float:
    """Device time of the dominant kernel of the last scan issued by this thread (needs set_timing)."""
    out = ctypes.c_float(0.0)
    check(lib().xfbq_last_scan_ms(ctypes.byref(out)))
    return float(out.value)


def scan_ms_mean() -> tuple[float, int]:
    """(mean device time of the dominant kernel, launches averaged) over the timed scans since set_timing(True)."""
    ms, cnt = ctypes.c_float(0.0), ctypes.c_int(0)
    check(lib().xfbq_scan_ms_mean(ctypes.byref(ms), ctypes.byref(cnt)))
    return float(ms.value), int(cnt.value)


def launch_count() -> int:
    return int(lib().xfbq_launch_count())


def require_cuda():
    """torch with a visible CUDA device, or a loud failure (never a host fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError(
            "no CUDA device visible: paper_2008_02002_b200 computes only on the GPU (no CPU fallback)")
    return torch
