"""The reference's .xfbq v1 index files (index.py:191-255): error classes on malformed files (host only),
and -- on the GPU -- files written by the unmodified reference load into the device layout, answer
k_select exactly like the reference did after its own load_index, and save back byte-identically.
Golden files: tests/golden/ref_index_*.xfbq + index_files.npz (oracle/gen_golden.py index-files)."""
import struct
from pathlib import Path

import numpy as np
import pytest

import paper_2008_02002_b200 as xb

GOLDEN = Path(__file__).resolve().parent / "golden"
HEADER = struct.Struct("<4sIIIBBdB")


def test_malformed_files_raise_the_reference_error_classes(tmp_path):
    """test_index.py:173-211: bad magic, truncated header, unsupported version, truncated payloads."""
    raw = (GOLDEN / "ref_index_with_originals.xfbq").read_bytes()
    magic, version, n, dim, wd, wq, scale, has = HEADER.unpack_from(raw)
    assert (magic, version, n, dim, wd, wq, has) == (b"XFBQ", 1, 96, 70, 3, 4, 1)
    p = tmp_path / "x.xfbq"
    p.write_bytes(b"NOPE" + raw[4:])
    with pytest.raises(xb.BadMagicError):
        xb.load_index(p)
    p.write_bytes(raw[:2])
    with pytest.raises(xb.BadMagicError):
        xb.load_index(p)
    p.write_bytes(raw[:HEADER.size - 3])
    with pytest.raises(xb.TruncatedIndexError):
        xb.load_index(p)
    p.write_bytes(HEADER.pack(b"XFBQ", 2, n, dim, wd, wq, scale, has) + raw[HEADER.size:])
    with pytest.raises(xb.UnsupportedVersionError):
        xb.load_index(p)
    p.write_bytes(raw[:HEADER.size + 100])
    with pytest.raises(xb.TruncatedIndexError):
        xb.load_index(p)
    plane_bytes = n * wd * 2 * 8
    p.write_bytes(raw[:HEADER.size + plane_bytes + 40])
    with pytest.raises(xb.TruncatedIndexError):
        xb.load_index(p)
    assert issubclass(xb.BadMagicError, xb.IndexFormatError) and issubclass(xb.IndexFormatError, xb.XfbqError)
    p.write_bytes(HEADER.pack(b"XFBQ", 1, n, dim, 9, wq, scale, has) + raw[HEADER.size:])
    with pytest.raises(xb.InvalidInputError):   # QuantParams validation, as in the reference
        xb.load_index(p)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["with_originals", "codes_only"])
def test_reference_files_load_search_and_round_trip(tag, tmp_path):
    z = np.load(GOLDEN / "index_files.npz")
    src = GOLDEN / f"ref_index_{tag}.xfbq"
    idx = xb.load_index(src)
    assert idx.params.scale == float(z[f"{tag}_scale"])
    assert np.array_equal(idx.packed.planes, z[f"{tag}_planes"])
    assert (idx.originals is not None) == (tag == "with_originals")
    for qi, q in enumerate(z[f"{tag}_queries"]):
        res = xb.k_select(idx, xb.SearchRequest(query=q, k=7, extra_distance=3))
        assert [h[0] for h in res.hits] == z[f"{tag}_ids"][qi].tolist()
        got = np.array([h[1] for h in res.hits])
        if tag == "with_originals":   # float64 refine: summation order differs, ids are exact
            assert np.allclose(got, z[f"{tag}_sims"][qi], rtol=0, atol=1e-12)
        else:
            assert got.tolist() == z[f"{tag}_sims"][qi].tolist()
        assert res.threshold_distance == int(z[f"{tag}_thr"][qi]) and res.candidate_count == int(z[f"{tag}_cand"][qi])
    out = tmp_path / "again.xfbq"
    xb.save_index(idx, out)
    assert out.read_bytes() == src.read_bytes()
    with pytest.raises(xb.InvalidInputError):
        xb.save_index(xb.Index(params=idx.params, packed=idx.packed, originals=None, ids=np.arange(idx.n)), out)
