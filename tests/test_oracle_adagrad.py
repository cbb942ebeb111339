"""The oracle's Adagrad restatement (a SELF-PINNED extension: the reference
has no Adagrad; BASELINE config 3 asks for its state in the
table). Pinned here against an independent numpy float32 restatement of the
published rule (Duchi et al. 2011, diagonal form):

    s <- s + g*g ;  v <- v - lr*g / (sqrt(s) + eps)

numpy float32 arithmetic and np.sqrt are IEEE correctly rounded, op by op,
like the C restatement (-ffp-contract=off) and the device's _rn intrinsics.
At train_reference level the first step from zero state is pinned against
the reference-pinned forward/backward gradient (or_forward_backward, checked
against oracle/_ref in test_oracle_golden.py)."""
import numpy as np

from native import make_cfg


def np_adagrad(v, s, g, lr, eps):
    v, s, g = (np.asarray(x, np.float32) for x in (v, s, g))
    lr, eps = np.float32(lr), np.float32(eps)
    s2 = (s + g * g).astype(np.float32)
    step = ((lr * g).astype(np.float32) / (np.sqrt(s2) + eps).astype(np.float32)).astype(np.float32)
    return (v - step).astype(np.float32), s2


def test_adagrad_step_matches_numpy_bitwise(oracle):
    rng = np.random.default_rng(0)
    for scale in (1e-6, 1e-2, 1.0, 1e3):
        v = rng.standard_normal(4096).astype(np.float32) * np.float32(scale)
        s = np.abs(rng.standard_normal(4096)).astype(np.float32) * np.float32(scale)
        g = rng.standard_normal(4096).astype(np.float32) * np.float32(scale)
        g[::7] = 0.0
        s[::11] = 0.0
        got_v, got_s = oracle.adagrad_apply(v, s, g, 0.05, 1e-8)
        want_v, want_s = np_adagrad(v, s, g, 0.05, 1e-8)
        assert got_v.tobytes() == want_v.tobytes()
        assert got_s.tobytes() == want_s.tobytes()


def test_adagrad_zero_gradient_leaves_row_and_state(oracle):
    v = np.array([1.5, -2.0, 0.0], np.float32)
    s = np.array([0.0, 4.0, 0.0], np.float32)
    got_v, got_s = oracle.adagrad_apply(v, s, np.zeros(3, np.float32), 0.05, 1e-8)
    assert np.array_equal(got_v, v) and np.array_equal(got_s, s)


def test_train_reference_first_adagrad_step(oracle, pkg):
    """One batch, one mini-batch, one device: rows = Adagrad step of the
    shard's mean gradient from zero embedding and zero state; state = g*g."""
    dims, B, E, layers = 3000, 256, 8, (8, 16, 1)
    off, keys, lab = pkg.gen_dataset(dims, B, 12, zipf=True, seed=4)
    cfg = make_cfg(1, 1, E, layers, J=1, optimizer="adagrad", eps=1e-8)
    dense, wk, wr = oracle.train_reference(cfg, B, off, keys, lab)
    assert wr.shape == (wk.size, 2 * E)
    w0 = oracle.init_dense(cfg)
    emb_keys = np.unique(keys)
    _, _, sg = oracle.forward_backward(E, layers, w0, off, keys, lab, emb_keys,
                                       np.zeros((emb_keys.size, E), np.float32))
    want_v, want_s = np_adagrad(np.zeros_like(sg), np.zeros_like(sg), sg, 0.05, 1e-8)
    assert np.array_equal(wk, emb_keys)
    assert wr[:, :E].tobytes() == want_v.tobytes()
    assert wr[:, E:].tobytes() == want_s.tobytes()
    # the dense path is the optimizer-independent SGD of the reference
    d_sgd, k_sgd, r_sgd = oracle.train_reference(make_cfg(1, 1, E, layers, J=1), B, off, keys,
                                                  lab)
    assert np.array_equal(dense, d_sgd)


def test_train_reference_adagrad_multi_device_canonical(oracle, pkg):
    """Four devices push their shard gradients; the owner applies them one
    sender at a time in canonical order. Differs from SGD, stays finite, and
    the state is a sum of squares (non-negative, non-decreasing)."""
    dims, B, E = 2000, 512, 4
    off, keys, lab = pkg.gen_dataset(dims, 3 * B, 10, zipf=True, seed=6)
    cfg = make_cfg(1, 4, E, (4, 1), J=2, optimizer="adagrad", eps=1e-6)
    _, wk, wr = oracle.train_reference(cfg, B, off, keys, lab)
    assert np.isfinite(wr).all()
    assert (wr[:, E:] >= 0).all() and (wr[:, E:] > 0).any()
    _, _, r_sgd = oracle.train_reference(make_cfg(1, 4, E, (4, 1), J=2), B, off, keys, lab)
    assert not np.array_equal(wr[:, :E], r_sgd)
