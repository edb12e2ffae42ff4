"""CPU oracle of the CNN model (oracle/cnn.c) against an independent float64 PyTorch
restatement: forward, loss, every parameter gradient, the SGD update, eval, and
the data / init conventions.  CPU only."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle_lib as ol

N_TRAIN, N_VAL = 1024, 256


@pytest.fixture(scope="module")
def ds():
    return ol.cnn_dataset(N_TRAIN, N_VAL)


def unpack(w):
    """Parameter vector -> float64 torch tensors (NCHW conv weights over the real channels)."""
    _, _, off = ol.cnn_layout()
    cin, creal, cout = (4, 32, 64), (3, 32, 64), (32, 64, 128)
    out = []
    for l in range(3):
        W = w[off[2 * l]: off[2 * l] + cout[l] * 9 * cin[l]].reshape(cout[l], 3, 3, cin[l])[..., :creal[l]]
        out.append(torch.tensor(W, dtype=torch.float64).permute(0, 3, 1, 2).contiguous().requires_grad_())
        out.append(torch.tensor(w[off[2 * l + 1]: off[2 * l + 1] + cout[l]], dtype=torch.float64).requires_grad_())
    out.append(torch.tensor(w[off[6]: off[6] + 16 * 128].reshape(16, 128)[:10], dtype=torch.float64).requires_grad_())
    out.append(torch.tensor(w[off[7]: off[7] + 10], dtype=torch.float64).requires_grad_())
    return out


def torch_loss(params, x, y):
    W1, b1, W2, b2, W3, b3, W4, b4 = params
    xt = torch.tensor(x.reshape(-1, 32, 32, 4)[..., :3], dtype=torch.float64).permute(0, 3, 1, 2)
    h = F.relu(F.conv2d(xt, W1, b1, stride=1, padding=1))
    h = F.relu(F.conv2d(h, W2, b2, stride=2, padding=1))
    h = F.relu(F.conv2d(h, W3, b3, stride=2, padding=1))
    g = h.mean(dim=(2, 3))
    z = g @ W4.T + b4
    return F.cross_entropy(z, torch.tensor(y, dtype=torch.long)), z


def grad_vector(params, like):
    _, _, off = ol.cnn_layout()
    cin, creal, cout = (4, 32, 64), (3, 32, 64), (32, 64, 128)
    g = np.zeros_like(like, dtype=np.float64)
    for l in range(3):
        G = np.zeros((cout[l], 3, 3, cin[l]))
        G[..., :creal[l]] = params[2 * l].grad.permute(0, 2, 3, 1).numpy()
        g[off[2 * l]: off[2 * l] + G.size] = G.ravel()
        g[off[2 * l + 1]: off[2 * l + 1] + cout[l]] = params[2 * l + 1].grad.numpy()
    G4 = np.zeros((16, 128))
    G4[:10] = params[6].grad.numpy()
    g[off[6]: off[6] + G4.size] = G4.ravel()
    g[off[7]: off[7] + 10] = params[7].grad.numpy()
    return g


def test_layout_and_init(ds):
    pa, pl, off = ol.cnn_layout()
    assert pa == 94538 and pl % 64 == 0 and off[8] <= pl
    s = ol.CnnSlot(ds)
    w = s.w.reshape(-1)
    W1 = w[: 32 * 36].reshape(32, 9, 4)
    assert np.all(W1[..., 3] == 0) and np.all(W1[..., :3] != 0).sum() > 0
    assert np.all(w[off[6] + 10 * 128: off[6] + 16 * 128] == 0)            # padded classifier rows
    for l, fan in enumerate((27, 288, 576)):
        W = w[off[2 * l]: off[2 * l + 1]]
        assert np.abs(W).max() <= np.sqrt(6 / fan) * (1 + 1e-6)
    assert not s.m.any()


def test_dataset_conventions(ds):
    x = ds.x.reshape(-1, 32, 32, 4)
    assert np.all(x[..., 3] == 0)
    assert np.all(np.abs(x * 128 - np.round(x * 128)) == 0) and x.min() >= -1 and x.max() < 1
    assert np.array_equal(ds.x[N_TRAIN:], ds.x[:256]) and np.array_equal(ds.y[N_TRAIN:], ds.y[:256])
    counts = np.bincount(ds.y[:N_TRAIN], minlength=10)
    assert (counts > 0).sum() >= 5


@pytest.mark.parametrize("B", [8, 21])
def test_one_step_gradient_vs_torch_float64(ds, B):
    s = ol.CnnSlot(ds, max_steps=4)
    w0 = s.w.copy()
    params = unpack(w0)
    loss, _ = torch_loss(params, ds.x[:B], ds.y[:B])
    loss.backward()
    g = grad_vector(params, w0)
    hp = np.tile(np.float32([1.0, 0.0, 0.0, B]), (4, 1))   # lr 1, mu 0, wd 0: m_1 = g, w_1 = w_0 - g
    s.train(hp, 1)
    assert abs(s.loss[0] - loss.item()) <= 2e-6 * abs(loss.item())
    _, _, off = ol.cnn_layout()
    for a, b in zip(off[:8], off[1:9]):
        ref, got = g[a:b], s.m[a:b].astype(np.float64)
        assert np.linalg.norm(got - ref) <= 1e-5 * np.linalg.norm(ref) + 1e-12, (a, b)
    assert np.array_equal(s.w, (w0 - s.m).astype(np.float32)) or np.allclose(s.w, w0 - s.m, atol=0)
    assert s.step.value == 1 and s.offset.value == B


def test_update_rule_momentum_wd(ds):
    s = ol.CnnSlot(ds, max_steps=4)
    hp = np.tile(np.float32([0.05, 0.9, 1e-3, 16]), (4, 1))
    s.train(hp, 1)
    w1, m1 = s.w.copy(), s.m.copy()
    s2 = ol.CnnSlot(ds, max_steps=4)
    s2.train(np.tile(np.float32([1.0, 0.0, 0.0, 16]), (4, 1)), 1)
    g = s2.m  # plain gradient at w0
    w0 = ol.CnnSlot(ds).w
    m_ref = np.fma(np.float32(0.9), np.float32(0), np.fma(np.float32(1e-3), w0, g)) if hasattr(np, "fma") else None
    # float64 check of g' = g + wd w ; m = g' ; w = w - lr m
    m64 = g.astype(np.float64) + 1e-3 * w0.astype(np.float64)
    assert np.allclose(m1, m64, rtol=1e-6, atol=1e-9)
    assert np.allclose(w1, w0 - np.float32(0.05) * m1, rtol=1e-6, atol=1e-9)
    del m_ref


def test_eval_vs_torch(ds):
    s = ol.CnnSlot(ds)
    vl, va = s.eval()
    params = unpack(s.w)
    with torch.no_grad():
        loss, z = torch_loss(params, ds.vx, ds.vy)
    assert abs(vl - loss.item()) <= 1e-5 * abs(loss.item())
    acc = (z.argmax(1).numpy() == ds.vy).mean()
    assert abs(va - acc) <= 1.5 / len(ds.vy)


def test_training_reduces_loss(ds):
    s = ol.CnnSlot(ds, max_steps=64)
    hp = np.tile(np.float32([0.05, 0.9, 1e-4, 32]), (64, 1))
    before = s.eval()[0]
    s.train(hp, 24)
    assert s.eval()[0] < before
    assert np.isfinite(s.loss[:24]).all()
