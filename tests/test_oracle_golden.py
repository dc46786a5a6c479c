"""Pin the CPU oracle (numpy and C restatements) to outputs of the unmodified reference.

Fixtures under tests/golden were written by oracle/gen_golden.py, which imports
/root/reference/pkg/src/xfbq in the build container.  Reference test citations are
paths under /root/reference/pkg/tests.
"""
import numpy as np
import pytest

from oracle import xfbq_oracle as xo
from tests._golden import SYNTH, load, sha, small_cases, synth_case


def test_quantize_values_golden_f64_all_widths():
    z = load("quant_values")
    xs = z["xs64"]
    for w in range(1, 9):
        assert np.array_equal(xo.np_quantize_values(xs, w), z[f"codes64_w{w}"])
        # C path through the f64 matrix entry
        planes = xo.c_quantize_matrix(xs[None, :], w, 1.0)
        assert np.array_equal(xo.np_unpack_codes(planes, xs.size)[0], z[f"codes64_w{w}"])


def test_quantize_values_golden_f32_scaled():
    z = load("quant_values")
    xs = z["xs32"]
    for w in range(1, 9):
        for si, s in enumerate(z["scales"]):
            want = z[f"codes32_w{w}_s{si}"]
            assert np.array_equal(xo.np_quantize_values(xs.astype(np.float64) * float(s), w), want)
            planes = xo.c_quantize_matrix(xs[None, :], w, float(s))
            assert np.array_equal(xo.np_unpack_codes(planes, xs.size)[0], want)


def test_worked_examples():
    # test_quant.py:74-87  0.3 -> 0b010, 0.0 -> 0b011, -0.999 -> 0b111 at 3 bits
    assert xo.np_quantize_values(np.array([0.3, 0.0, -0.999]), 3).tolist() == [0b010, 0b011, 0b111]
    # test_quant.py:114-118 saturation
    assert xo.np_quantize_values(np.array([1.0, 1.5, 100.0]), 4).tolist() == [0, 0, 0]
    assert xo.np_quantize_values(np.array([-1.0, -2.5, -1e9]), 4).tolist() == [15, 15, 15]
    # test_bitplane.py:27-32 bit transpose of codes [010, 111]
    p = xo.np_pack_code_matrix(np.array([[0b010, 0b111]], dtype=np.uint8), 3)
    assert [int(p[b, 0, 0]) for b in (2, 1, 0)] == [0b10, 0b11, 0b10]
    # test_bitplane.py:116-123 quantize_vector composes scaling
    pv = xo.np_quantize_vector(np.array([0.3, -0.999]), 3, 1.0)
    assert [int(pv[b, 0]) for b in (2, 1, 0)] == [0b10, 0b11, 0b10]
    z = load("worked")
    # test_search.py:129-144 distances [20, 17, 26, 17, 23]
    planes = xo.np_quantize_matrix(z["pipeline_values"], 3, 1.0)
    q = xo.np_quantize_vector(np.array([0.375]), 3, 1.0)
    assert xo.np_batch_distances(planes, q).tolist() == [20, 17, 26, 17, 23]
    assert xo.c_batch_distances(planes, q).tolist() == z["pipeline_dists"].tolist()
    d, i = xo.np_topk(z["pipeline_dists"], 2)
    assert i.tolist() == [1, 3] and d.tolist() == [17, 17]  # tie broken by id
    # test_distance.py:30-35  55 / 40
    x = xo.np_pack_code_matrix(np.array([[0b010, 0b010]], dtype=np.uint8), 3)
    y = xo.np_pack_code_matrix(np.array([[0b010, 0b111]], dtype=np.uint8), 3)
    assert int(xo.np_batch_distances(x, y[:, :, 0])[0]) == 55
    assert int(xo.np_batch_distances(x, x[:, :, 0])[0]) == 40
    assert z["pd_xy"].tolist() == [55, 40]
    # test_distance.py:86-89
    assert [xo.distance_upper_bound(200, 3, 4), xo.distance_upper_bound(0, 3, 4),
            xo.distance_upper_bound(64, 3, 3)] == z["ub"].tolist() == [21000, 0, 3136]


def test_small_cases_numpy_and_c():
    count = 0
    for c in small_cases():
        planes_np = xo.np_quantize_matrix(c["docs"], c["wd"], c["scale"])
        planes_c = xo.c_quantize_matrix(c["docs"], c["wd"], c["scale"])
        assert np.array_equal(planes_np, c["planes"]), c["ci"]
        assert np.array_equal(planes_c, c["planes"]), c["ci"]
        qp_np = np.stack([xo.np_quantize_vector(q, c["wq"], c["scale"]) for q in c["queries"]])
        qp_c = xo.c_quantize_matrix(c["queries"], c["wq"], c["scale"]).transpose(2, 0, 1)
        assert np.array_equal(qp_np, c["qplanes"])
        assert np.array_equal(qp_c, c["qplanes"])
        for qi in range(c["nq"]):
            assert np.array_equal(xo.np_batch_distances(c["planes"], c["qplanes"][qi]), c["full"][qi])
            assert np.array_equal(xo.c_batch_distances(c["planes"], c["qplanes"][qi]), c["full"][qi])
        d_np, i_np = xo.np_search(c["planes"], c["qplanes"], c["k"])
        d_c, i_c = xo.c_search(c["planes"], c["qplanes"], c["k"], threads=2)
        assert np.array_equal(d_np, c["dists"]) and np.array_equal(i_np, c["ids"])
        assert np.array_equal(d_c, c["dists"]) and np.array_equal(i_c, c["ids"])
        # decoded similarities equal k_select's hits (search.py:167-171)
        sims = xo.np_decode_inner_product_values(c["dists"], c["dim"], c["wd"], c["wq"])
        sims /= c["scale"] * c["scale"]
        assert np.array_equal(sims, c["sims"])
        count += 1
    assert count == 84


@pytest.mark.parametrize("name", SYNTH)
def test_synthetic_cases_c_oracle(name):
    c = synth_case(name)
    z = c["z"]
    planes = xo.c_quantize_matrix(c["docs"], c["wd"], c["scale"])
    assert sha(planes) == str(z["planes_sha"])
    assert np.array_equal(planes[:, :, :64], z["planes_head"])
    assert np.array_equal(planes[:, :, -64:], z["planes_tail"])
    qplanes = xo.c_quantize_matrix(c["queries"].astype(np.float64), c["wq"], c["scale"]).transpose(2, 0, 1)
    d, i = xo.c_search(planes, qplanes, c["k"])
    assert np.array_equal(d, z["dists"])
    assert np.array_equal(i, z["ids"])
    # row_offset shifts ids only
    d2, i2 = xo.c_search(planes, qplanes[:2], c["k"], row_offset=1000, threads=1)
    assert np.array_equal(d2, z["dists"][:2]) and np.array_equal(i2, z["ids"][:2] + 1000)


def test_estimate_scale_matches_reference():
    c = synth_case("cfg4_40k_256_w4")
    assert xo.estimate_scale(c["docs"][:1_000_000], 0.98) == c["scale"]


def test_numpy_oracle_on_one_synthetic_case():
    c = synth_case("cfg3_50k_200_w4")
    z = c["z"]
    sub = 3000  # numpy restatement is slow: check a prefix of rows for planes, one query for top-k
    planes = xo.np_quantize_matrix(c["docs"][:sub], c["wd"], c["scale"])
    full = xo.c_quantize_matrix(c["docs"], c["wd"], c["scale"])
    assert np.array_equal(planes, full[:, :, :sub])
    q = xo.np_quantize_vector(c["queries"][0].astype(np.float64), c["wq"], c["scale"])
    d = xo.np_batch_distances(full, q)
    dd, ii = xo.np_topk(d, c["k"])
    assert np.array_equal(dd, z["dists"][0]) and np.array_equal(ii, z["ids"][0])


def test_edge_cases():
    # k > n returns n hits; n == 0 returns nothing (test_search.py:205-215)
    planes = xo.np_quantize_matrix(np.zeros((3, 5), dtype=np.float32), 3, 1.0)
    q = xo.np_quantize_vector(np.zeros(5), 4, 1.0)[None]
    d, i = xo.c_search(planes, q, 10)
    assert d.shape == (1, 3) and i.tolist() == [[0, 1, 2]]
    empty = np.zeros((3, 1, 0), dtype=np.uint64)
    d, i = xo.c_search(empty, q, 10)
    assert d.shape == (1, 0)
    with pytest.raises(ValueError):
        xo.np_quantize_values(np.array([0.1, np.nan]), 3)
    with pytest.raises(ValueError):
        xo.c_quantize_matrix(np.array([[0.1, np.inf]], dtype=np.float32), 3, 1.0)


def test_bench_corpus_generator_is_the_reference_recipe():
    """bench.py's corpus chunks (both arms) = generate_synthetic's recipe (dataio.py:104-124), which
    synthetic_unit_rows restates and the golden hashes above pin to the reference's own output."""
    import bench
    for c, rows, dim in ((0, 1000, 256), (3, 257, 200)):
        assert np.array_equal(bench.gen_chunk_host(c, rows, dim), xo.synthetic_unit_rows(rows, dim, 4000 + c))
    got = []
    bench.gen_rows_host(5, 2_000_050, 3_000_000, 8, lambda first, x: got.append((first, x.shape[0])), workers=2)
    assert got == [(5, 999_995), (1_000_000, 1_000_000), (2_000_000, 50)]
