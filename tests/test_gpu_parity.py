"""GPU parity tests: the CUDA path (through the Python drop-in API -> ctypes -> C ABI) against
the golden outputs of the unmodified reference (tests/golden, oracle/gen_golden.py) and against
the CPU oracle on the same seeded inputs.  Integer/byte/index work: bit-exact.

Reference test citations are paths under /root/reference/pkg/tests.
"""
import os
import warnings

import numpy as np
import pytest

import paper_2008_02002_b200 as xb
from oracle import xfbq_oracle as xo
from tests._golden import SYNTH, load, sha, small_cases, synth_case

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _quiet():
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        yield


def _codes_of(packed):
    return xb.unpack_matrix(packed)


# ------------------------------------------------------------------ quantizer (kernel 1)
def test_quantize_values_golden_f64_all_widths():
    z = load("quant_values")
    xs = z["xs64"]
    for w in range(1, 9):
        pm = xb.quantize_matrix(xs[None, :], w, 1.0)
        assert np.array_equal(_codes_of(pm)[0], z[f"codes64_w{w}"]), w
        # row-major many-rows form too (each value its own row, dim 1)
        pm = xb.quantize_matrix(xs[:, None], w, 1.0)
        assert np.array_equal(_codes_of(pm)[:, 0], z[f"codes64_w{w}"]), w


def test_quantize_values_golden_f32_scaled():
    """float32 input widened in-kernel to float64 then scaled (bitplane.py:229-232), including
    denormals, +-0, saturating values and grid neighbours (test_quant.py:132-143)."""
    z = load("quant_values")
    xs = z["xs32"]
    assert xs.dtype == np.float32
    for w in range(1, 9):
        for si, s in enumerate(z["scales"]):
            pm = xb.quantize_matrix(xs[None, :], w, float(s))
            assert np.array_equal(_codes_of(pm)[0], z[f"codes32_w{w}_s{si}"]), (w, si)


def test_worked_examples():
    # test_quant.py:74-87 / test_bitplane.py:116-123
    pv = xb.quantize_vector(np.array([0.3, -0.999]), 3, 1.0)
    assert [int(pv.planes[b, 0]) for b in (2, 1, 0)] == [0b10, 0b11, 0b10]
    assert _codes_of(xb.quantize_matrix(np.array([[0.3, 0.0, -0.999]]), 3))[0].tolist() == [0b010, 0b011, 0b111]
    # test_quant.py:114-118 saturation
    assert _codes_of(xb.quantize_matrix(np.array([[1.0, 1.5, 100.0]]), 4))[0].tolist() == [0, 0, 0]
    assert _codes_of(xb.quantize_matrix(np.array([[-1.0, -2.5, -1e9]]), 4))[0].tolist() == [15, 15, 15]
    z = load("worked")
    # test_search.py:129-155: distances [20, 17, 26, 17, 23], tie broken by id
    params = xb.QuantParams(dim=1, scale=1.0, doc_bits=3, query_bits=3)
    idx = xb.build_index(z["pipeline_values"], params, keep_originals=False)
    d = xb.batch_distances(idx.packed, xb.quantize_vector(np.array([0.375]), 3, 1.0))
    assert d.dtype == np.uint64 and d.tolist() == [20, 17, 26, 17, 23]
    scores, ids = xb.search(idx, np.array([[0.375]]), 2)
    assert scores.tolist() == [[17, 17]] and ids.tolist() == [[1, 3]]
    res = xb.k_select(idx, xb.SearchRequest(query=np.array([0.375]), k=2))
    assert [h[0] for h in res.hits] == [1, 3] and res.approximate
    assert res.threshold_distance == 17 and res.candidate_count == 2
    # test_distance.py:30-35  55 / 40
    x = xb.pack_matrix(np.array([[0b010, 0b010]], dtype=np.uint8), 3)
    y = xb.pack_matrix(np.array([[0b010, 0b111]], dtype=np.uint8), 3)
    assert int(xb.batch_distances(x, y.row(0))[0]) == 55
    assert int(xb.batch_distances(x, x.row(0))[0]) == 40


def test_small_cases_everything_bit_exact():
    """84 ragged cases: dims {1..513} x widths {(3,4),(4,4),(8,8),(1,8),(2,1),(5,3)}: planes,
    query planes, full distances, top-k (with exact ties), decoded sims, threshold, candidates."""
    count = 0
    for c in small_cases():
        params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
        idx = xb.build_index(c["docs"], params, keep_originals=False)
        assert np.array_equal(idx.packed.planes, c["planes"]), c["ci"]
        assert idx.packed.nbytes == c["planes"].nbytes
        for qi in range(c["nq"]):
            pq = xb.quantize_vector(c["queries"][qi], c["wq"], c["scale"])
            assert np.array_equal(pq.planes, c["qplanes"][qi]), (c["ci"], qi)
            assert np.array_equal(xb.batch_distances(idx.packed, pq), c["full"][qi]), (c["ci"], qi)
        scores, ids = xb.search(idx, c["queries"], c["k"])
        assert scores.shape == c["dists"].shape
        assert np.array_equal(scores.astype(np.uint64), c["dists"]), c["ci"]
        assert np.array_equal(ids, c["ids"]), c["ci"]
        res = xb.k_select(idx, xb.SearchRequest(query=c["queries"][0], k=c["k"]))
        assert [h[0] for h in res.hits] == c["ids"][0].tolist()
        assert [h[1] for h in res.hits] == c["sims"][0].tolist()
        assert res.threshold_distance == int(c["thr"][0]) and res.candidate_count == int(c["cand"][0])
        # a PackedMatrix rebuilt from reference planes scans identically (layout conversion)
        pm = xb.PackedMatrix(c["planes"], c["dim"])
        idx2 = xb.Index(params=params, packed=pm, originals=None)
        s2, i2 = xb.search(idx2, c["queries"], c["k"])
        assert np.array_equal(s2, scores) and np.array_equal(i2, ids)
        count += 1
    assert count == 84


@pytest.mark.parametrize("name", SYNTH)
def test_synthetic_configs_match_reference(name):
    """Config-shaped synthetic corpora (reference generator, seeds in the fixture): packed planes
    hash, top-k distances and ids for every query equal the unmodified reference's."""
    c = synth_case(name)
    z = c["z"]
    params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
    idx = xb.build_index(c["docs"], params, keep_originals=False)
    planes = idx.packed.planes
    assert sha(planes) == str(z["planes_sha"])
    assert np.array_equal(planes[:, :, :64], z["planes_head"])
    scores, ids = xb.search(idx, c["queries"], c["k"])
    assert np.array_equal(scores.astype(np.uint64), z["dists"])
    assert np.array_equal(ids, z["ids"])
    # float64 queries give the same answer (float32 -> float64 is exact)
    s64, i64 = xb.search(idx, c["queries"].astype(np.float64), c["k"])
    assert np.array_equal(s64, scores) and np.array_equal(i64, ids)
    for qi in (0, c["nq"] - 1):
        res = xb.k_select(idx, xb.SearchRequest(query=c["queries"][qi], k=c["k"]))
        assert [h[0] for h in res.hits] == z["ids"][qi].tolist()
        assert [h[1] for h in res.hits] == z["sims"][qi].tolist()
        assert res.threshold_distance == int(z["thr"][qi]) and res.candidate_count == int(z["cand"][qi])


@pytest.mark.parametrize("env", [{"XFBQ_FORCE_GENERIC": "1"}, {"XFBQ_GRID": "1"}, {"XFBQ_GRID": "7"},
                                 {"XFBQ_SAMPLE": "0"}, {"XFBQ_SAMPLE": "2048"}, {"XFBQ_SAMPLE": "2048", "XFBQ_GRID": "3"},
                                 {"XFBQ_ENGINE": "popc"}, {"XFBQ_ENGINE": "popc", "XFBQ_TQ": "1"},
                                 {"XFBQ_ENGINE": "popc", "XFBQ_TQ": "5", "XFBQ_SPLITS": "3"},
                                 {"XFBQ_ENGINE": "imma"}, {"XFBQ_ENGINE": "umma"}, {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE": "0"},
                                 {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_SLICES": "7"}, {"XFBQ_ENGINE": "umma", "XFBQ_SAMPLE": "0"},
                                 {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_STAGES": "2", "XFBQ_GRID": "5"}])
def test_scan_plans_agree(env, monkeypatch):
    """Every launch plan (generic/specialised kernel, query-tile size, document splits) yields the
    same keys: the order on (distance, id) is total, so the result is partition independent."""
    c = synth_case("cfg4_40k_256_w4")
    z = c["z"]
    params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
    idx = xb.build_index(c["docs"], params, keep_originals=False)
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    scores, ids = xb.search(idx, c["queries"], c["k"])
    assert np.array_equal(scores.astype(np.uint64), z["dists"]) and np.array_equal(ids, z["ids"])


@pytest.mark.parametrize("name,nq,k", [("cfg4_40k_256_w4", 700, 100), ("cfg2_60k_128_w3", 300, 10),
                                       ("cfg3_50k_200_w4", 520, 33), ("cfg5_20k_512_w4", 150, 1000)])
def test_batch_mode_many_queries(name, nq, k):
    """Enough queries to fill whole CTAs of the batch plan (8 query warps per CTA, several query
    groups, several document splits); every query checked against the CPU oracle."""
    c = synth_case(name)
    params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
    idx = xb.build_index(c["docs"], params, keep_originals=False)
    queries = xo.synthetic_unit_rows(nq, c["dim"], 777)
    scores, ids = xb.search(idx, queries, k)
    planes = xo.c_quantize_matrix(c["docs"], c["wd"], c["scale"])
    qp = xo.c_quantize_matrix(queries.astype(np.float64), c["wq"], c["scale"]).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, k)
    assert np.array_equal(scores.astype(np.uint64), want_d) and np.array_equal(ids, want_i)


@pytest.mark.parametrize("engine", ["umma", "imma"])
@pytest.mark.parametrize("n,dim,wd,nq,k", [(5000, 256, 4, 40, 10), (33333, 128, 3, 130, 7), (12345, 200, 4, 257, 33),
                                           (9000, 512, 4, 150, 100), (3000, 100, 4, 20, 1000), (40000, 64, 2, 600, 1),
                                           (70000, 256, 4, 1000, 100)])
def test_tensor_engines_ragged_shapes(engine, n, dim, wd, nq, k, monkeypatch):
    """Both tensor engines (tcgen05 with TMEM accumulators / mma.sync IMMA) on ragged shapes: n not a multiple of
    the 128-document stage, dims that pad to 128, every (C, query-tile) kernel variant, k from 1 to 1000; every
    query against the CPU oracle."""
    docs = xo.synthetic_unit_rows(n, dim, 11 + n)
    queries = xo.synthetic_unit_rows(nq, dim, 12 + n)
    scale = xo.estimate_scale(docs, 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4)
    idx = xb.build_index(docs, params, keep_originals=False)
    monkeypatch.setenv("XFBQ_ENGINE", engine)
    scores, ids = xb.search(idx, queries, k)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, k)
    assert np.array_equal(scores.astype(np.uint64), want_d) and np.array_equal(ids, want_i)


@pytest.mark.parametrize("generic", [False, True])
def test_collect_candidates_matches_distance_array(generic, monkeypatch):
    """The one-pass candidate gather of k_select (count + row ids of d <= threshold, no distance array) against
    the materialised distances, for thresholds from 'nothing' to 'everything'; a small id buffer forces the
    second pass."""
    import torch
    from paper_2008_02002_b200.distance import batch_distances_device, collect_candidates_device
    c = synth_case("cfg3_50k_200_w4")
    params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
    idx = xb.build_index(c["docs"], params, keep_originals=False)
    upper = xb.distance_upper_bound(c["dim"], c["wd"], c["wq"])
    if generic:
        monkeypatch.setenv("XFBQ_FORCE_GENERIC", "1")  # the any-width kernel instead of the <WD, WQ, C> specialisation
    for qi in (0, 3):
        pq = xb.quantize_vector(c["queries"][qi], c["wq"], c["scale"])
        d = batch_distances_device(idx.packed, pq)
        srt = torch.sort(d).values
        for thr in (-1, 0, int(srt[0]) - 1, int(srt[0]), int(srt[9]), int(srt[999]), int(srt[-1]), upper):
            count, ids = collect_candidates_device(idx.packed, pq, thr, want_ids=True, cap=16)
            want = torch.nonzero(d <= thr).flatten()
            assert count == want.numel()
            assert torch.equal(torch.sort(ids).values, want)
            count_only, none = collect_candidates_device(idx.packed, pq, thr, want_ids=False)
            assert count_only == count and none is None


_SEEDED = {"XFBQ_ENGINE": "umma", "XFBQ_UMMA_QUEUE_MIN_N": "1", "XFBQ_SAMPLE": "4096"}


@pytest.mark.parametrize("extra", [{}, {"XFBQ_SEED_BELOW4": "0"}, {"XFBQ_SEED_BELOW4": "40"}, {"XFBQ_MERGE_BOUNDED": "0"},
                                   {"XFBQ_SEED_HIST": "0"}, {"XFBQ_UMMA_SLICES": "3", "XFBQ_GRID": "9"},
                                   {"XFBQ_UMMA_SHARE": "0"}, {"XFBQ_UMMA_HIST": "0"},
                                   {"XFBQ_MERGE_BUF": "256", "XFBQ_UMMA_SLICES": "6", "XFBQ_SEED_BELOW4": "0"}])
@pytest.mark.parametrize("n,dim,wd,nq,k", [(70000, 256, 4, 1000, 100), (70001, 128, 3, 600, 10), (80000, 512, 4, 300, 50)])
def test_counted_seed_queue_scan_and_bounded_merge(extra, n, dim, wd, nq, k, monkeypatch):
    """The route full-size batches take, forced onto a corpus the CPU oracle can check: thresholds seeded by
    counting the sample's scores into per-query histograms, the queue kernel over document slices with the
    shared candidate histogram, and the merge that drops keys beyond the proven bound.  The variants move the
    histogram frame to where it misses for many queries (open thresholds) or catches everything in the last
    bin, and switch each piece back to its predecessor: thresholds only ever prune, the keys never change."""
    docs = xo.synthetic_unit_rows(n, dim, 21 + n)
    queries = xo.synthetic_unit_rows(nq, dim, 22 + n)
    scale = xo.estimate_scale(docs, 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4)
    idx = xb.build_index(docs, params, keep_originals=False)
    for key, val in {**_SEEDED, **extra}.items():
        monkeypatch.setenv(key, val)
    scores, ids = xb.search(idx, queries, k)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, k)
    assert np.array_equal(scores.astype(np.uint64), want_d) and np.array_equal(ids, want_i)


@pytest.mark.parametrize("extra", [{}, {"XFBQ_SEED_BELOW4": "0"}, {"XFBQ_SEED_BELOW4": "40"}, {"XFBQ_SEED_HIST": "0"}])
@pytest.mark.parametrize("n,dim,wd,nq,k", [(70000, 256, 4, 1, 100), (70001, 128, 3, 5, 10), (80000, 512, 4, 16, 50),
                                           (66000, 200, 4, 2, 1000)])
def test_small_batches_counted_seed(extra, n, dim, wd, nq, k, monkeypatch):
    """Small batches (mma.sync engine, the documents split over every warp of the chip) take their thresholds from
    the counting kernel of the tcgen05 path; frames that miss or catch everything, and the list-keeping sample scan
    it replaced, give the same keys."""
    docs = xo.synthetic_unit_rows(n, dim, 31 + n)
    queries = xo.synthetic_unit_rows(nq, dim, 32 + n)
    scale = xo.estimate_scale(docs, 0.98)
    params = xb.QuantParams(dim=dim, scale=scale, doc_bits=wd, query_bits=4)
    idx = xb.build_index(docs, params, keep_originals=False)
    for key, val in {"XFBQ_SAMPLE": "4096", **extra}.items():
        monkeypatch.setenv(key, val)
    scores, ids = xb.search(idx, queries, k)
    planes = xo.c_quantize_matrix(docs, wd, scale)
    qp = xo.c_quantize_matrix(queries.astype(np.float64), 4, scale).transpose(2, 0, 1)
    want_d, want_i = xo.c_search(planes, qp, k)
    assert np.array_equal(scores.astype(np.uint64), want_d) and np.array_equal(ids, want_i)


@pytest.mark.parametrize("width", [1, 2, 3, 4, 5, 6, 7, 8])
def test_fast_float32_quantizer_on_code_boundaries(width, monkeypatch):
    """The float32-first quantizer (exact float64 redo near code boundaries) against the CPU oracle and the
    all-float64 kernel: values on and up to 40 ulps around every code boundary, saturation edges, denormals, +-0,
    huge values, zero-heavy rows, plus random data; dims that leave a ragged last float4 group of a lane."""
    import torch
    rng = np.random.default_rng(100 + width)
    for scale in (1.0, 0.7310585786300049, 3.3333333333333335, 12.345, 1e-3):
        half = 2.0 ** (width - 1)
        g32 = (np.arange(-half - 3, half + 4) / (scale * half)).astype(np.float32)
        up = np.nextafter(g32, np.float32(np.inf))
        dn = np.nextafter(g32, np.float32(-np.inf))
        special = np.array([0.0, -0.0, 1e-45, -1e-45, 1e-38, -1e-38, 3e38, -3e38, 1.0, -1.0, 0.5, -0.5], dtype=np.float32)
        rnd = rng.uniform(-2, 2, size=6000).astype(np.float32) / np.float32(scale)
        # every float32 within 40 ulps of a boundary: the fast path's window (+-1024 of 2^32 integers over the clip range) is
        # 8-16 ulps wide at the outer boundaries, so both its edges and its inside are covered
        bits = g32.view(np.int32)[None, :] + np.arange(-40, 41, dtype=np.int32)[:, None]
        sweep = bits.astype(np.int32).view(np.float32).ravel()
        sweep = sweep[np.isfinite(sweep)]
        sparse = rnd[:2000] * (rng.random(2000) < 0.3)   # zero-heavy rows: x = 0 sits exactly on a boundary
        vals = np.concatenate([g32, up, dn, np.nextafter(up, np.float32(np.inf)), np.nextafter(dn, np.float32(-np.inf)), special, rnd,
                               sweep, sparse.astype(np.float32)])
        dim = 200                                   # ragged: the fourth lane of a row holds 8 of its 32 dims
        vals = np.concatenate([vals, np.zeros((-len(vals)) % dim, np.float32)]).reshape(-1, dim).astype(np.float32)
        want = xo.c_quantize_matrix(vals, width, scale)
        monkeypatch.delenv("XFBQ_QUANT_SLOW", raising=False)
        fast = xb.quantize_matrix(torch.from_numpy(vals).cuda(), width, scale).planes
        monkeypatch.setenv("XFBQ_QUANT_SLOW", "1")
        slow = xb.quantize_matrix(torch.from_numpy(vals).cuda(), width, scale).planes
        assert np.array_equal(fast, want) and np.array_equal(slow, want), (width, scale)
    monkeypatch.delenv("XFBQ_QUANT_SLOW", raising=False)
    with pytest.raises(xb.InvalidInputError):       # non-finite values are still caught (quant.py:142-143)
        xb.quantize_matrix(torch.tensor([[1.0, float("inf"), 0.0, 0.0]], device="cuda"), width, 1.0)
    with pytest.raises(xb.InvalidInputError):
        xb.quantize_matrix(torch.tensor([[float("nan"), 0.0, 0.0, 0.0]], device="cuda"), width, 1.0)
    for bad in (float("inf"), float("-inf"), float("nan")):   # anywhere in a row, among ordinary values
        rows = rng.uniform(-1, 1, size=(70, 256)).astype(np.float32)
        rows[33, 157] = bad
        with pytest.raises(xb.InvalidInputError):
            xb.quantize_matrix(torch.from_numpy(rows).cuda(), width, 1.0)


def test_concurrent_searches_are_deterministic():
    """test_search.py:254-265: searches from a thread pool on one shared index give exactly the serial answers
    (the library keeps no global mutable state: thread-local error string / timing, caller-owned workspaces)."""
    from concurrent.futures import ThreadPoolExecutor
    c = synth_case("cfg4_40k_256_w4")
    z = c["z"]
    params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
    idx = xb.build_index(c["docs"], params, keep_originals=False)
    batches = [xo.synthetic_unit_rows(96, c["dim"], 4242 + j) for j in range(3)]   # tcgen05 engine; DIFFERENT queries per batch:
    serial_batch = [xb.search(idx, b, 50) for b in batches]                          # threads that shared a workspace would mix them up
    serial_single = [xb.k_select(idx, xb.SearchRequest(query=q, k=c["k"])) for q in c["queries"][:8]]

    def work(i):
        if i % 2:
            return xb.search(idx, batches[(i // 2) % 3], 50)
        return xb.k_select(idx, xb.SearchRequest(query=c["queries"][(i // 2) % 8], k=c["k"]))

    with ThreadPoolExecutor(max_workers=8) as pool:
        results = list(pool.map(work, range(96)))
    for i, r in enumerate(results):
        if i % 2:
            want = serial_batch[(i // 2) % 3]
            assert np.array_equal(r[0], want[0]) and np.array_equal(r[1], want[1]), i
        else:
            want = serial_single[(i // 2) % 8]
            assert r.hits == want.hits and r.threshold_distance == want.threshold_distance, i
    assert [h[0] for h in serial_single[0].hits] == z["ids"][0].tolist()


def test_edge_cases():
    """k > n, empty index, dim mismatch, non-finite, bad scale (test_search.py:205-222,
    test_distance.py:143-153)."""
    params = xb.QuantParams(dim=5, scale=1.0, doc_bits=3, query_bits=4)
    idx = xb.build_index(np.zeros((3, 5), dtype=np.float32), params, keep_originals=False)
    scores, ids = xb.search(idx, np.zeros((2, 5)), 10)
    assert scores.shape == (2, 3) and ids.tolist() == [[0, 1, 2], [0, 1, 2]]
    res = xb.k_select(idx, xb.SearchRequest(query=np.zeros(5), k=10))
    assert len(res.hits) == 3
    empty = xb.build_index(np.zeros((0, 5), dtype=np.float32), params, keep_originals=False)
    assert empty.n == 0
    s, i = xb.search(empty, np.zeros((2, 5)), 4)
    assert s.shape == (2, 0)
    res = xb.k_select(empty, xb.SearchRequest(query=np.zeros(5), k=3))
    assert res.hits == [] and res.candidate_count == 0 and res.threshold_distance == 0
    assert xb.batch_distances(empty.packed, xb.quantize_vector(np.zeros(5), 4)).shape == (0,)
    with pytest.raises(xb.DimensionMismatchError):
        xb.search(idx, np.zeros((1, 6)), 1)
    with pytest.raises(xb.DimensionMismatchError):
        xb.k_select(idx, xb.SearchRequest(query=np.zeros(6), k=1))
    with pytest.raises(xb.DimensionMismatchError):
        xb.batch_distances(idx.packed, xb.quantize_vector(np.zeros(6), 4))
    with pytest.raises(xb.InvalidInputError):
        xb.batch_distances(idx.packed, xb.quantize_vector(np.zeros(5), 4), out=np.zeros(4, dtype=np.uint64))
    with pytest.raises(xb.InvalidInputError):
        xb.build_index(np.array([[0.1, np.inf, 0, 0, 0]], dtype=np.float32), params)
    with pytest.raises(xb.InvalidInputError):
        xb.quantize_matrix(np.array([[1e300, 1.0]]), 3, 1e300)  # scaled value overflows to inf
    with pytest.raises(xb.InvalidInputError):
        xb.search(idx, np.zeros((1, 5)), 0)
    # non-finite queries raise whether they arrive from the host (check read after the scan is enqueued), from
    # pinned memory or from the device (check read right after the quantizer): quant.py:142-143
    import torch
    bad_q = np.array([[0.0, np.nan, 0.0, 0.0, 0.0], [0.0, 0.0, 0.0, 0.0, 0.0]])
    for q in (bad_q, bad_q.astype(np.float32), torch.from_numpy(bad_q).pin_memory(), torch.from_numpy(bad_q).cuda()):
        with pytest.raises(xb.InvalidInputError):
            xb.search(idx, q, 2)
    s_ok, i_ok = xb.search(idx, torch.zeros((2, 5), dtype=torch.float64).pin_memory(), 2)
    assert i_ok.tolist() == [[0, 1], [0, 1]]
    with pytest.raises(xb.InvalidInputError):
        xb.PackedMatrix(np.full((3, 1, 2), 1 << 40, dtype=np.uint64), 5)  # padding bits set


def test_k_select_with_originals_and_external_ids():
    """Full pipeline with float refine (search.py:153-157): same ids as the CPU composition,
    sims to 1e-12 (float64 summation order differs between BLAS and the GPU)."""
    c = synth_case("cfg3_50k_200_w4")
    params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
    ext = np.arange(c["n"], dtype=np.int64) * 3 + 7
    idx = xb.build_index(c["docs"], params, ids=ext)
    planes = xo.c_quantize_matrix(c["docs"], c["wd"], c["scale"])
    docs64 = c["docs"].astype(np.float64)
    for qi in range(4):
        q = c["queries"][qi].astype(np.float64)
        extra = 300
        res = xb.k_select(idx, xb.SearchRequest(query=q, k=10, extra_distance=extra), collect_timing=True)
        d = xo.c_batch_distances(planes, xo.np_quantize_vector(q, c["wq"], c["scale"]))
        thr = int(np.sort(d)[9]) + extra
        cand = np.flatnonzero(d <= thr)
        sims = docs64[cand] @ q
        order = np.lexsort((cand, -sims))[:10]
        assert res.threshold_distance == thr and res.candidate_count == cand.size and not res.approximate
        assert [h[0] for h in res.hits] == ext[cand[order]].tolist()
        assert np.allclose([h[1] for h in res.hits], sims[order], rtol=0, atol=1e-12)
        assert set(res.stage_seconds) == {"quantize_query", "distances", "histogram_gather", "refine"}


def test_merge_topk_kernel_against_numpy():
    import torch
    from paper_2008_02002_b200 import _native
    L = _native.lib()
    rng = np.random.default_rng(5)
    for parts, nq, k in [(1, 3, 1), (2, 5, 10), (8, 4, 100), (37, 2, 1000), (300, 3, 100), (3, 2, 4096)]:
        raw = rng.integers(0, 1 << 40, size=(parts, nq, k), dtype=np.uint64)
        raw[rng.random(raw.shape) < 0.1] = np.uint64(0xFFFFFFFFFFFFFFFF)
        raw.sort(axis=2)
        dev = torch.from_numpy(raw.view(np.int64)).cuda()
        out = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        _native.check(L.xfbq_merge_topk(dev.data_ptr(), parts, nq, k, out.data_ptr(), 0))
        torch.cuda.synchronize()
        want = np.sort(raw.transpose(1, 0, 2).reshape(nq, parts * k), axis=1)[:, :k]
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (parts, nq, k)


def test_large_k_and_sharded_equals_single():
    """top-1000 (config-5 shaped) and the multi-GPU composition on one device: shards scanned with
    row offsets then merged equal the single scan equal the reference."""
    import torch
    from paper_2008_02002_b200 import _native
    from paper_2008_02002_b200.search import scan_topk_device, unpack_keys_device
    c = synth_case("cfg5_20k_512_w4")
    z = c["z"]
    params = xb.QuantParams(dim=c["dim"], scale=c["scale"], doc_bits=c["wd"], query_bits=c["wq"])
    idx = xb.build_index(c["docs"], params, keep_originals=False)
    scores, ids = xb.search(idx, c["queries"], c["k"])
    assert np.array_equal(scores.astype(np.uint64), z["dists"]) and np.array_equal(ids, z["ids"])
    L = _native.lib()
    G = 3
    per = -(-c["n"] // G)
    qwords = xb.quantize_queries(c["queries"], c["wq"], c["scale"])
    parts = []
    for g in range(G):
        lo, hi = g * per, min(c["n"], (g + 1) * per)
        shard = xb.quantize_matrix(c["docs"][lo:hi], c["wd"], c["scale"])
        parts.append(scan_topk_device(shard, qwords, c["nq"], c["wq"], c["k"], row_offset=lo))
    stacked = torch.stack(parts).contiguous()
    out = torch.empty_like(parts[0])
    _native.check(L.xfbq_merge_topk(stacked.data_ptr(), G, c["nq"], c["k"], out.data_ptr(), 0))
    d, i = unpack_keys_device(out)
    assert np.array_equal(d.cpu().numpy().astype(np.uint64), z["dists"]) and np.array_equal(i.cpu().numpy(), z["ids"])
