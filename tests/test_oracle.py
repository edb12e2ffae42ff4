"""CPU oracle self-checks (no GPU): deterministic transcendental functions, synthetic data,
init, and the training arithmetic against an independent numpy restatement."""
import math

import numpy as np
import pytest

from oracle_lib import D0, Dataset, Slot, dataset, layout, oracle


def test_layout():
    p_algo, p_alloc, off = layout()
    assert p_algo == 784 * 256 + 256 + 256 * 256 + 256 + 10 * 256 + 10
    assert off == [0, 200704, 200960, 266496, 266752, 270848, 270864]
    assert p_alloc % 64 == 0 and p_alloc >= off[6]


def test_exp_det_accuracy():
    lib = oracle()
    xs = np.concatenate([-np.linspace(0, 87, 20001, dtype=np.float32), np.float32([-1e-8, -0.5, -86.99])])
    worst = 0.0
    for x in xs:
        got = lib.orc_exp(float(x))
        want = math.exp(float(x))
        worst = max(worst, abs(got - want) / want)
    assert worst < 4e-7  # a few ulp
    assert lib.orc_exp(-90.0) == 0.0 and lib.orc_exp(0.0) == 1.0


def test_log_det_accuracy():
    lib = oracle()
    xs = np.concatenate([np.linspace(1, 10, 20001, dtype=np.float32), np.float32([1.0000001, 1.41421, 1.41422, 2, 4])])
    worst = 0.0
    for x in xs:
        got = lib.orc_log(float(x))
        want = math.log(float(np.float32(x)))
        worst = max(worst, abs(got - want))
    assert worst < 4e-7
    assert lib.orc_log(1.0) == 0.0


def test_dataset_properties_and_determinism():
    ds = dataset()
    x, y = ds.x, ds.y
    assert x.shape == (65536 + 256, D0)
    k = x * 128
    assert np.all(k == np.round(k)) and k.min() >= -128 and k.max() <= 127
    # wrap rows duplicate the head so any window of <= max_batch samples is contiguous
    assert np.array_equal(x[65536:], x[:256]) and np.array_equal(y[65536:], y[:256])
    counts = np.bincount(y[:65536], minlength=10)
    assert counts.min() > 1000  # every class present
    assert Dataset().digest() == ds.digest()
    assert not np.array_equal(ds.vx[:16], x[:16])


def test_init_is_he_uniform_and_pads_zero():
    p_algo, p_alloc, off = layout()
    s = Slot()
    w = s.w
    assert np.all(s.m == 0)
    w1 = w[off[0]:off[1]]
    bound = math.sqrt(6 / 784)
    assert np.abs(w1).max() <= bound and np.abs(w1).max() > 0.99 * bound
    assert np.all(w[off[1]:off[2]] == 0)  # b1
    assert np.all(w[off[4] + 10 * 256:off[5]] == 0)  # W3 padding rows
    assert np.all(w[off[6]:] == 0)


def np_step(w, m, hp, x, y, off):
    """float64-free numpy restatement of one step (float32, fused ops emulated in float64 then rounded)."""
    lr, mu, wd, bs = (float(v) for v in hp)
    B = int(bs)
    f32 = np.float32
    W1 = w[off[0]:off[1]].reshape(256, 784)
    b1 = w[off[1]:off[2]]
    W2 = w[off[2]:off[3]].reshape(256, 256)
    b2 = w[off[3]:off[4]]
    W3 = w[off[4]:off[5]].reshape(16, 256)
    b3 = w[off[5]:off[6]]
    X = x[:B].astype(np.float64)
    h1 = np.maximum(X @ W1.T + b1, 0)
    h2 = np.maximum(h1 @ W2.T + b2, 0)
    z = h2 @ W3.T + b3
    zz = z[:, :10] - z[:, :10].max(1, keepdims=True)
    p = np.exp(zz) / np.exp(zz).sum(1, keepdims=True)
    loss = float(np.mean(-np.log(p[np.arange(B), y[:B]])))
    dz = p.copy()
    dz[np.arange(B), y[:B]] -= 1
    dz /= B
    dz16 = np.zeros((B, 16))
    dz16[:, :10] = dz
    g = np.zeros_like(w, dtype=np.float64)
    g[off[4]:off[5]] = (dz16.T @ h2).ravel()
    g[off[5]:off[6]] = dz16.sum(0)
    dh2 = (dz16 @ W3) * (h2 > 0)
    g[off[2]:off[3]] = (dh2.T @ h1).ravel()
    g[off[3]:off[4]] = dh2.sum(0)
    dh1 = (dh2 @ W2) * (h1 > 0)
    g[off[0]:off[1]] = (dh1.T @ X).ravel()
    g[off[1]:off[2]] = dh1.sum(0)
    m2 = mu * m + (g + wd * w)
    w2 = w - lr * m2
    return w2.astype(f32), m2.astype(f32), loss


def test_train_step_matches_float64_restatement():
    """The oracle's fp32 training step agrees with a float64 numpy restatement to fp32 accuracy
    (checks the arithmetic *definition*, independently of rounding details)."""
    _, _, off = layout()
    ds = dataset()
    s = Slot()
    hp = np.tile(np.float32([0.1, 0.9, 1e-3, 128]), (8, 1))
    w, m = s.w.astype(np.float64), s.m.astype(np.float64)
    offset = 0
    for step in range(3):
        s.train(hp, 1)
        w_ref, m_ref, loss_ref = np_step(w, m, hp[step], ds.x[offset:], ds.y[offset:], off)
        assert abs(s.loss[step] - loss_ref) < 1e-5 * max(1, loss_ref)
        np.testing.assert_allclose(s.w, w_ref, rtol=2e-4, atol=2e-6)
        np.testing.assert_allclose(s.m, m_ref, rtol=2e-3, atol=2e-6)
        w, m = s.w.astype(np.float64), s.m.astype(np.float64)
        offset += 128
    assert s.step.value == 3 and s.offset.value == 384


def test_loss_decreases_and_eval_improves():
    s = Slot()
    hp = np.tile(np.float32([0.05, 0.9, 0.0, 128]), (200, 1))
    l0, a0 = s.eval()
    s.train(hp, 200)
    l1, a1 = s.eval()
    assert s.loss[:10].mean() > s.loss[190:200].mean()
    assert l1 < l0 and a1 > a0 + 0.1


def test_oracle_is_deterministic_and_resumable():
    """Training 40 steps == training 15 then 25 (stage splitting is invisible)."""
    hp = np.tile(np.float32([0.1, 0.5, 1e-4, 64]), (40, 1))
    hp[20:, 3] = 128  # batch-size change mid-run
    a = Slot()
    a.train(hp, 40)
    b = Slot()
    b.train(hp, 15)
    c = b.copy()
    c.train(hp, 25)
    assert np.array_equal(a.w, c.w) and np.array_equal(a.m, c.m)
    assert np.array_equal(a.loss[:40], c.loss[:40])
    assert a.offset.value == 20 * 64 + 20 * 128


def test_train_rejects_short_hp_table():
    s = Slot()
    with pytest.raises(AssertionError):
        s.train(np.tile(np.float32([0.1, 0.9, 0, 32]), (2, 1)), 3)
