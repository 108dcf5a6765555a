"""GPU parity on edge cases: erasures (LLR 0), saturated LLRs, isolated and
degree-1 nodes, edge-free codes, odd gamma, I = 1 streams, large gamma."""
import numpy as np
import pytest

from oracle import bp as obp
from oracle import qc as oqc
from oracle import stream as ost

pytestmark = pytest.mark.gpu
TOL = 1e-4


def close(got, ref):
    err = np.abs(np.asarray(got) - np.asarray(ref)) / np.maximum(np.abs(ref), 1.0)
    assert err.max() <= TOL, err.max()


def same_decode(q, rows, n, mu, iters, early=False):
    lay = q.build_edge_layout(q.SparseParityCheck(n, rows))
    olay = oqc.layout_from_rows(n, rows)
    r = q.decode_llr_batch(lay, mu, iters, early_stop=early)
    bits, post, ok, its = obp.decode_llr(olay, mu, iters, early_stop=early)
    assert np.array_equal(r.hard_bits, bits)
    assert np.array_equal(r.syndrome_ok, ok)
    assert np.array_equal(r.iterations_run, its)
    close(r.posteriors, post)
    return r


def test_erasures_and_saturation(gpu):
    q = gpu
    exp = q.multiplicative_shifts(3, 6, 7)
    h = q.expand_qc(exp)
    rng = np.random.default_rng(4)
    mu = rng.normal(2.0, 2.5, size=(37, h.n))
    mu[:, ::5] = 0.0                     # erasures
    mu[3] = 0.0                          # an all-erased lane
    mu[4, :10] = 1e6                     # clipped to +50
    mu[5, :10] = -1e6
    same_decode(q, h.rows, h.n, mu, 15)
    same_decode(q, h.rows, h.n, mu, 15, early=True)


def test_isolated_and_degree_one_nodes(gpu):
    q = gpu
    rows = [[0], [1, 2], [2, 3, 4], [0, 4, 6]]      # variable 5 in no check, check 0 degree 1
    rng = np.random.default_rng(6)
    mu = rng.normal(1.0, 1.5, size=(9, 7))
    r = same_decode(q, rows, 7, mu, 6)
    assert np.allclose(r.posteriors[:, 5], np.clip(mu[:, 5], -50, 50), atol=1e-5)


def test_code_without_edges(gpu):
    q = gpu
    lay = q.build_edge_layout(q.SparseParityCheck(4, [[], []]))
    mu = np.array([[1.0, -2.0, 0.5, -0.1]])
    r = q.decode_llr_batch(lay, mu, 3)
    assert r.hard_bits.tolist() == [[0, 1, 0, 1]] and r.syndrome_ok.all()


@pytest.mark.parametrize("G", [1, 2, 31, 33, 65, 100])
def test_odd_gamma(gpu, G):
    q = gpu
    exp = q.multiplicative_shifts(2, 4, 8)
    h = q.expand_qc(exp)
    mu = np.random.default_rng(G).normal(1.5, 2.0, size=(G, h.n))
    same_decode(q, h.rows, h.n, mu, 9)


def test_large_gamma_large_code(gpu):
    q = gpu
    h, exp = q.load_code(q.codes.bundled_code_path("code_d_like"))
    lay = q.build_edge_layout(h)
    G = 1024
    sigma = q.ebn0_to_sigma(3.0, 5 / 6)
    y = q.simulate_block(q.ChannelConfig(3.0, 5 / 6, seed=2, gamma=G), lay.n_vars)
    r = q.decode_batch(lay, y, sigma, 20)
    # check a sample of lanes against the oracle (float64 on the CPU)
    olay = oqc.qc_layout(exp.shifts, exp.p)
    pick = np.array([0, 1, 511, 1023])
    bits, post, ok, _ = obp.decode_llr(olay, obp.channel_llrs(y[pick], sigma), 20)
    assert np.array_equal(r.hard_bits[pick], bits) and np.array_equal(r.syndrome_ok[pick], ok)


def test_stream_single_processor(gpu):
    q = gpu
    code = q.unwrap_qc(q.multiplicative_shifts(4, 8, 5))
    U = oqc.unwrap(oqc.array_code_shifts(4, 8, 5), 5)
    rng = np.random.default_rng(12)
    ys = rng.normal(1.0, 0.9, size=(9, 2, code.c))
    dec, odec = q.StreamDecoder(code, 1, gamma=2), ost.StreamOracle(U, 1, 2)
    out = [f for f in (dec.push_frame(y, 0.9) for y in ys) if f] + dec.flush()
    ref = [f for f in (odec.push(y, 0.9) for y in ys) if f] + odec.flush()
    assert [f.frame_index for f in out] == [f.frame_index for f in ref] == list(range(9))
    for a, b in zip(out, ref):
        assert np.array_equal(a.hard_bits, b.hard_bits)
        close(a.posteriors, b.posteriors)
