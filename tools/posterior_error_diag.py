import sys, numpy as np
sys.path.insert(0, '.')
import paper_1204_0334_b200 as q
from oracle import bp as obp, qc as oqc
for (J, L, p, G) in [(3, 6, 31, 128), (3, 12, 29, 96), (2, 8, 37, 64), (4, 16, 23, 256)]:
    exp = q.multiplicative_shifts(J, L, p)
    lay = q.build_edge_layout(q.expand_qc(exp))
    olay = oqc.qc_layout(exp.shifts, p)
    y = np.random.default_rng(J * 100 + L).normal(1.0, 0.75, size=(G, lay.n_vars))
    for it in (1, 3, 8, 15):
        r = q.decode_batch(lay, y, 0.75, it)
        bits, post, ok, its = obp.decode_llr(olay, obp.channel_llrs(y, 0.75), it)
        err = np.abs(r.posteriors - post) / np.maximum(np.abs(post), 1.0)
        i = np.unravel_index(err.argmax(), err.shape)
        print(J, L, p, it, "max", f"{err.max():.2e}", "p99.99", f"{np.quantile(err, 0.9999):.2e}", "at post", f"{post[i]:.4f}", "gpu", f"{r.posteriors[i]:.4f}", "bits_eq", np.array_equal(r.hard_bits, bits))
