"""CPU: host-side logic (code model, plans' inputs, bit packing, stop rule, codegen)."""
import io

import numpy as np
import pytest
from conftest import golden

import paper_1204_0334_b200 as q
from oracle import qc as oqc
from paper_1204_0334_b200 import codegen
from paper_1204_0334_b200.dist import ordered_prefix
from paper_1204_0334_b200.plan import lane_words, unpack_planes


def test_edge_layout_matches_oracle(codes_npz):
    for sh, p in ((oqc.array_code_shifts(2, 4, 8), 8), (codes_npz["code_a_shifts"], 422)):
        lay = q.build_edge_layout(q.expand_qc(q.ExponentMatrix(sh, p)))
        o = oqc.qc_layout(sh, p)
        assert np.array_equal(lay.check_pad, o.check_pad)
        assert np.array_equal(lay.var_pad, o.var_pad)
        assert np.array_equal(lay.edge_var, o.edge_var)
        assert lay.check_regular == o.check_pad.shape[1]


def test_worked_example_tables():
    lay = q.build_edge_layout(q.SparseParityCheck(8, [[1, 3, 4, 7], [0, 1, 2, 5], [2, 5, 6, 7], [0, 3, 4, 6]]))
    assert [lay.check_edges(m).tolist() for m in range(4)] == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11], [12, 13, 14, 15]]
    assert [v.tolist() for v in lay.var_edges] == [[4, 12], [0, 5], [6, 8], [1, 13], [2, 14], [7, 9], [10, 15], [3, 11]]


def test_irregular_padding():
    lay = q.build_edge_layout(q.SparseParityCheck(5, [[0, 1, 2], [2, 3], [0, 4]]))
    assert lay.check_regular is None
    assert lay.check_pad.tolist() == [[0, 1, 2], [3, 4, 7], [5, 6, 7]]


def test_unwrapped_tables(codes_npz):
    code = q.unwrap_qc(q.ExponentMatrix(codes_npz["code_a_shifts"], 422))
    o = oqc.unwrap(codes_npz["code_a_shifts"], 422)
    assert (code.lam, code.ms, code.c, code.cb, code.edge_count) == (4, 3, 2532, 422, 40512)
    assert np.array_equal(code.lut_c, o.lut_c) and np.array_equal(code.lut_v, o.lut_v)
    assert np.array_equal(code.sub_offset, o.sub_offset)
    assert code.rate_bound == pytest.approx(5 / 6) and code.period == 4
    with pytest.raises(ValueError):
        q.unwrap_qc(q.multiplicative_shifts(3, 5, 7))


def test_qc_file_roundtrip(tmp_path, codes_npz):
    exp = q.ExponentMatrix(codes_npz["code_a_shifts"], 422)
    path = str(tmp_path / "a.qc")
    q.save_code(path, q.expand_qc(exp), exp)
    h, e2 = q.load_code(path)
    assert np.array_equal(e2.shifts, exp.shifts) and h == q.expand_qc(exp)
    small = q.expand_qc(q.multiplicative_shifts(2, 4, 5))
    ap = str(tmp_path / "s.alist")
    q.save_code(ap, small)
    h2, none = q.load_code(ap)
    assert none is None and h2 == small
    assert np.array_equal(q.infer_qc_structure(small).shifts, q.multiplicative_shifts(2, 4, 5).shifts)
    bad = tmp_path / "b.qc"
    bad.write_text("2 3 5\n0 1 2\n")
    with pytest.raises(q.CodeFormatError):
        q.load_code(str(bad))


@pytest.mark.parametrize("name,p,seed", [("n18360", 765, 18360), ("code_b_like", 632, 632),
                                         ("code_c_like", 768, 768), ("code_d_like", 1024, 1024)])
def test_bundled_codes_are_girth8_and_reproducible(name, p, seed):
    h, exp = q.load_code(q.codes.bundled_code_path(name))
    assert (h.n, h.m, exp.edge_count) == (24 * p, 4 * p, 96 * p)
    assert not codegen.has_short_cycles(exp.shifts, exp.p)
    assert np.array_equal(codegen.girth8_shifts(4, 24, p, seed=seed), exp.shifts)


def test_lane_words_roundtrip():
    rng = np.random.default_rng(0)
    a = rng.random(70) < 0.5
    w = lane_words(a, 96)
    assert w.shape == (3,)
    bits = unpack_planes(w[None, :], 70)[0]
    assert np.array_equal(bits.astype(bool), a)
    assert (w[0] >> 3) & 1 == a[3]


def test_ordered_prefix_stop_rule():
    rows = [(8, 3, 1), (8, 0, 0), (8, 9, 2), (8, 1, 1)]
    tot, done, used = ordered_prefix(rows, stop_errors=3, max_frames=1000)
    assert done and used == 3 and tot == (24, 12, 3)
    tot, done, used = ordered_prefix(rows[:2], stop_errors=3, max_frames=1000)
    assert not done and tot == (16, 3, 1)
    tot, done, used = ordered_prefix(rows[2:], 3, 1000, tot)
    assert done and tot == (24, 12, 3)
    tot, done, used = ordered_prefix(rows, 100, 16)
    assert done and tot[0] == 16


def test_config_and_rows():
    cfg = q.SimulationConfig("x", 3.0)
    assert cfg.points() == [3.0] and q.SimulationConfig("x", [1, 2]).points() == [1.0, 2.0]
    r = q.PointResult("c", "block", 3.2, 30, 32, 64, 5, 1, 5 / (64 * 10), 1 / 64, 1.5, 42.6667, 100.0)
    assert r.row()[2] == "3.2" and r.row()[10] == "1.500"
    buf = io.StringIO()
    q.write_csv([r], buf)
    assert buf.getvalue().splitlines()[0].split(",") == q.CSV_COLUMNS
    with pytest.raises(ValueError):
        q.ChannelConfig(3.0, 0.0, seed=0)
    assert q.ebn0_to_sigma(3.2, 5 / 6) == pytest.approx(0.53588996575190975146, abs=1e-15)
