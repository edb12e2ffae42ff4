"""CNN model on the GPU (SMX_MODEL_CNN) against the CPU oracle (oracle/cnn.c):

* exact mode: dataset, init, multi-step trajectories (lr / momentum / wd / batch-size changes),
  loss history and eval metrics are bit-identical to the oracle;
* tensor-core mode (implicit-GEMM tcgen05 convolutions, 3xTF32): first-step loss and every
  gradient within the stated tolerance, short trajectories within the fp32 envelope, results
  grouping-invariant and run-to-run deterministic (bitwise);
* the engine runs a merged CNN study whose metrics equal the oracle's (exact mode).
"""
import json

import numpy as np
import pytest

import oracle_lib as ol
from paper_2006_11972_b200 import executor as ex
from paper_2006_11972_b200 import host
from test_cnn_oracle import grad_vector, torch_loss, unpack

pytestmark = pytest.mark.gpu

N_TRAIN, N_VAL, MAXB = 4096, 256, 64


@pytest.fixture(scope="module")
def ds():
    return ol.cnn_dataset(N_TRAIN, N_VAL, MAXB)


def make(mode, slots=4, ckpts=2, max_steps=64):
    return ex.Executor(n_slots=slots, n_ckpts=ckpts, gemm_mode=mode, max_steps=max_steps, max_batch=MAXB,
                       n_train=N_TRAIN, n_val=N_VAL, model=ex.MODEL_CNN)


def schedule(n, bs0=16, bs1=24):
    hp = np.zeros((n, 4), np.float32)
    for i in range(n):
        hp[i] = [0.05 if i < n // 2 else 0.02, 0.9 if i % 3 else 0.5, 1e-4 if i < n // 3 else 1e-3,
                 bs0 if i < n // 2 else bs1]
    return hp


def test_dataset_and_init_match_oracle(ds):
    with make(ex.GEMM_EXACT) as e:
        assert e.p_algo == 94538
        assert e.dataset_digest() == ds.digest()
        e.slot_init(1)
        w, m = e.slot_read(1)
        o = ol.CnnSlot(ds)
        assert np.array_equal(w, o.w) and not m.any()


def test_exact_trajectory_bitwise(ds):
    n = 6
    hp = schedule(n)
    with make(ex.GEMM_EXACT) as e:
        e.slot_init(0)
        e.hp_upload(0, 0, hp)
        e.train([0], n)
        w, m = e.slot_read(0)
        loss = e.losses(0, 0, n)
        met = tuple(e.eval([0])[0])
        step, off = e.slot_state(0)
    o = ol.CnnSlot(ds, max_steps=n + 1)
    o.train(hp, n)
    assert step == n and off == o.offset.value
    assert np.array_equal(loss, o.loss[:n])
    assert np.array_equal(w, o.w) and np.array_equal(m, o.m)
    assert met == o.eval()


def test_exact_grouping_and_save_load(ds):
    hp = schedule(4)
    with make(ex.GEMM_EXACT) as e:
        for s in range(3):
            e.slot_init(s)
            e.hp_upload(s, 0, hp if s != 1 else schedule(4, 32, 8))
        e.train([0, 1, 2], 2)
        e.slot_save(0, 0)
        e.train([0, 1, 2], 2)
        e.slot_load(2, 0)           # slot 2 restarts from slot 0's step-2 checkpoint
        e.hp_upload(2, 0, hp)
        e.train([2], 2)
        w0, m0 = e.slot_read(0)
        w2, m2 = e.slot_read(2)
    assert np.array_equal(w0, w2) and np.array_equal(m0, m2)


def rel(a, b):
    return np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30)


def check_first_step(ds, bs, maxb=MAXB, chan_bound=2e-5, n_val=N_VAL):
    """One tensor-core step at batch size bs (mu = 0: m_1 = the gradient) against the fp32 oracle's
    loss and a float64 torch gradient."""
    _, _, off = ol.cnn_layout()
    hp = np.tile(np.float32([1.0, 0.0, 0.0, bs]), (4, 1))
    with ex.Executor(n_slots=4, n_ckpts=2, gemm_mode=ex.GEMM_TC, max_steps=64, max_batch=maxb, n_train=N_TRAIN,
                     n_val=n_val, model=ex.MODEL_CNN) as e:
        e.slot_init(0)
        e.hp_upload(0, 0, hp)
        e.train([0], 1)
        _, m = e.slot_read(0)
        loss = e.losses(0, 0, 1)[0]
    o = ol.CnnSlot(ds, max_steps=4)
    w0 = o.w.copy()
    o.train(hp, 1)
    assert abs(loss - o.loss[0]) <= 2e-6 * abs(o.loss[0])
    # float64 ground truth: long reductions (up to bs x 1024 terms with cancellation) make the
    # fp32 oracle itself ~1e-4 off for conv1; the TC path must be as good as fp32 is
    params = unpack(w0)
    tl, _ = torch_loss(params, ds.x[:bs], ds.y[:bs])
    tl.backward()
    g64 = grad_vector(params, w0)
    # A pre-activation within ~1e-7 of 0 can flip its ReLU mask between any two fp32 evaluation
    # orders (measured: conv1 channel 14 at bs 16 flips for TC, at bs 64 for the oracle itself),
    # which moves that output channel's gradient by ~1e-3 relative.  The bound is therefore per
    # output channel: 90% of channels within 2e-5 (or twice the fp32 oracle's own error where that
    # is larger), every tensor within 2e-3.
    cout = (32, 32, 64, 64, 128, 128, 16, 16)
    for i, (a, b) in enumerate(zip(off[:8], off[1:9])):
        assert rel(m[a:b], g64[a:b]) <= 2e-3, (bs, i, rel(m[a:b], g64[a:b]))
        rows = [r for r in np.split(np.arange(a, b), cout[i]) if np.linalg.norm(g64[r]) > 0]
        errs = sorted(rel(m[r], g64[r]) for r in rows)
        oerrs = sorted(rel(o.m[r], g64[r]) for r in rows)
        bound = max(chan_bound, 2 * oerrs[int(0.9 * (len(oerrs) - 1))])
        assert errs[int(0.9 * (len(errs) - 1))] <= bound, (bs, i, errs[-3:], bound)


@pytest.mark.parametrize("bs", [1, 5, 16, 37, 64])
def test_tc_first_step_gradient(ds, bs):
    # bs 1 / 5 / 37: batch sizes that are not multiples of the conv1 weight-gradient work item
    # (4 samples) and of the 8 image-row chunks, and batches smaller than one item
    check_first_step(ds, bs)


@pytest.mark.parametrize("bs", [37, 1])
def test_tc_first_step_gradient_odd_max_batch(bs):
    # max_batch 37 (n_val a multiple of it and of 128): the conv3 input gradient's last M tile holds one
    # sample, and at bs 37 its second TMA output box sample (37) is past max_batch, so the tensor
    # store is clipped (kTmD2)
    check_first_step(ol.cnn_dataset(N_TRAIN, 128 * 37, 37), bs, maxb=37, n_val=128 * 37)


@pytest.mark.parametrize("bs", [200, 256])
def test_tc_first_step_gradient_max_batch_256(bs):
    # The largest batch (C3's bs 256 step): 8 weight-gradient splits of 2,048 rows for conv2, a
    # partial last split at bs 200, 64 conv1 work items per slot.  At this size the weight
    # gradients of conv1 / conv2 (bs x 1024 / bs x 256 terms per weight) are dominated by ReLU-mask
    # flips of their input activations: pre-activations within the forward's rounding of 0 change
    # mask between any two fp32 orders, and their number grows with bs.  Measured 90th-percentile
    # channel errors vs float64 at bs 200 / 256: fp32 oracle 2-6e-6, tensor-core path 2.9-4.2e-5
    # (segmenting the conv1 forward's TMEM accumulation 5 ways did not change this, swapping its
    # tcgen05 forward for fp32 FMA chains halved it).  Per-channel bound here: 1e-4 (tf32 alone
    # would be ~1e-3); every tensor still within 2e-3.
    check_first_step(ol.cnn_dataset(N_TRAIN, N_VAL, 256), bs, maxb=256, chan_bound=1e-4)


def test_tc_trajectory_and_eval_within_tolerance(ds):
    n = 20
    hp = schedule(n)
    with make(ex.GEMM_TC) as e:
        e.slot_init(0)
        e.hp_upload(0, 0, hp)
        e.train([0], n)
        w, _ = e.slot_read(0)
        loss = e.losses(0, 0, n)
        vl, va = e.eval([0])[0]
    o = ol.CnnSlot(ds, max_steps=n + 1)
    o.train(hp, n)
    assert np.max(np.abs(loss - o.loss[:n]) / np.abs(o.loss[:n])) <= 1e-4
    assert rel(w, o.w) <= 1e-3   # ReLU-boundary flips (see above) amplified over 20 steps: 1.4e-4 measured
    ovl, ova = o.eval()
    assert abs(vl - ovl) <= 1e-4 * abs(ovl) and abs(va - ova) <= 2 / N_VAL


def test_tc_grouping_invariance_and_determinism(ds):
    hp = schedule(3)
    outs = []
    for group in ([0], [0, 1, 2, 3], [3, 0]):
        with make(ex.GEMM_TC) as e:
            for s in range(4):
                e.slot_init(s)
                e.hp_upload(s, 0, hp if s == 0 else schedule(3, 64, 40))
            e.train(group, 3)
            outs.append((*e.slot_read(0), e.losses(0, 0, 3), tuple(e.eval([0])[0])))
    for o in outs[1:]:
        assert all(np.array_equal(a, b) for a, b in zip(o[:3], outs[0][:3])) and o[3] == outs[0][3]


def test_engine_cnn_study_exact_vs_oracle(ds):
    spec = json.dumps({
        "schema": 1, "name": "cnn_mini", "model": "cnn", "max_steps": 6,
        "space": {"lr": [{"family": "step", "initial": "0.05", "gamma": "0.1", "milestones": [3]},
                         {"family": "constant", "value": "0.05"}],
                  "batch_size": [{"family": "constant", "value": 16}]},
        "sampler": {"kind": "grid"}})
    e = host.Engine.for_study(spec, slots_per_gpu=2, max_batch=MAXB, n_train=N_TRAIN, n_val=N_VAL, gemm_mode=0)
    e.submit_study(spec)
    e.run()
    st = e.stats()
    assert st["stage_steps"] == 9 and st["trial_steps"] == 12
    info = host.expand_study(spec)
    from test_engine_gpu import hp_table
    for (study, trial), hist in e.histories().items():
        o = ol.CnnSlot(ds, max_steps=8)
        o.train(hp_table(info["trials"][trial]), 6)
        assert [(s, l, a) for s, l, a in hist] == [(6, *o.eval())]


def test_tc_determinism_many_slots(ds):
    """Run-to-run bitwise determinism at a full active set (64 slots, mixed batch sizes): many
    CTAs per kernel and a deep TMA ring, where a released-too-early operand slot shows up as
    differing gradients (profiles/debug/race_probe.py is the longer version)."""
    del ds
    ref = None
    for _ in range(3):
        with ex.Executor(n_slots=64, n_ckpts=2, gemm_mode=ex.GEMM_TC, max_steps=8, max_batch=128, n_train=8192,
                         n_val=256, model=ex.MODEL_CNN) as e:
            for s in range(64):
                e.slot_init(s)
                e.hp_upload(s, 0, np.tile(np.float32([0.05, 0.9, 1e-4, 128 if s % 2 == 0 else 64]), (8, 1)))
            e.train(list(range(64)), 1)
            ms = [e.slot_read(s)[1].copy() for s in range(64)]
        if ref is None:
            ref = ms
        else:
            bad = [s for s in range(64) if not np.array_equal(ms[s], ref[s])]
            assert not bad, f"slots with run-to-run differences: {bad}"
