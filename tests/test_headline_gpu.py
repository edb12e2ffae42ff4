"""Parity at the headline configuration (BASELINE configs[1] = C2, the bench's workload): the
CNN in tensor-core mode with max_batch 128, n_train 65,536, 64 slots grouped in one launch,
each slot with its own hp row at bs 128 — the exact shapes the 64-trial study runs.

Tolerances:
  * first-step loss |rel| <= 2e-6 against the fp32 oracle;
  * first-step update m_1 = g + wd w_0 of every slot against float64 (PyTorch): every parameter
    tensor rel-L2 <= 2e-3 and 90 % of its output channels <= 2e-5 (a pre-activation within
    ~1e-7 of zero flips its ReLU mask between any two fp32 orders);
  * 20-step bs-128 trajectories: per-step loss |rel| <= 1e-4, weights rel-L2 <= 1e-3, eval
    loss |rel| <= 1e-4 against the oracle;
  * uploaded N(0,1) data (not tf32-exact) takes the full 3xTF32 path: same first-step bounds
    (MLP §3.6: loss 2e-6, update 2e-5).
"""
import numpy as np
import pytest

import oracle_lib as ol
from paper_2006_11972_b200 import executor as ex
from test_cnn_oracle import grad_vector, torch_loss, unpack

pytestmark = pytest.mark.gpu

N_TRAIN, N_VAL, MAXB, SLOTS = 65536, 256, 128, 64
COUT = (32, 32, 64, 64, 128, 128, 16, 16)


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(np.asarray(b, np.float64)), 1e-30))


def c2_rows(n_slots):
    """64 distinct C2-style hp rows: lr {0.1, 0.05, 0.02, 0.01} x mu {0.9, 0.5, 0} x wd {5e-4, 1e-3, 0}."""
    rows = []
    for s in range(n_slots):
        rows.append([(0.1, 0.05, 0.02, 0.01)[s % 4], (0.9, 0.5, 0.0)[(s // 4) % 3], (5e-4, 1e-3, 0.0)[(s // 12) % 3],
                     128.0])
    return np.float32(rows)


@pytest.fixture(scope="module")
def ds():
    return ol.cnn_dataset(N_TRAIN, N_VAL, MAXB)


def cnn_exec(**kw):
    return ex.Executor(n_slots=SLOTS, n_ckpts=2, gemm_mode=ex.GEMM_TC, max_steps=kw.pop("max_steps", 32),
                       max_batch=MAXB, n_train=N_TRAIN, n_val=N_VAL, model=ex.MODEL_CNN, **kw)


def check_update(m, w0, wd, g64, off, tag):
    """m (fp32 first-step momentum = g + wd w0) against float64, per parameter tensor / channel."""
    ref = g64 + np.float64(wd) * w0.astype(np.float64)
    for i, (a, b) in enumerate(zip(off[:8], off[1:9])):
        r = rel(m[a:b], ref[a:b])
        assert r <= 2e-3, (tag, i, r)
        rows = [q for q in np.split(np.arange(a, b), COUT[i]) if np.linalg.norm(ref[q]) > 0]
        errs = sorted(rel(m[q], ref[q]) for q in rows)
        assert errs[int(0.9 * (len(errs) - 1))] <= 2e-5, (tag, i, errs[-3:])


def test_headline_first_step_64_slots(ds):
    """(i) 64 slots x bs 128 in one grouped launch, 64 distinct hp rows: first-step loss and every
    slot's update within tolerance of the fp32 oracle / float64."""
    rows = c2_rows(SLOTS)
    _, _, off = ol.cnn_layout()
    with cnn_exec() as e:
        for s in range(SLOTS):
            e.slot_init(s)
            e.hp_upload(s, 0, np.tile(rows[s], (4, 1)))
        e.train(list(range(SLOTS)), 1)
        got = [(e.losses(s, 0, 1)[0], *e.slot_read(s)) for s in range(SLOTS)]
    o = ol.CnnSlot(ds, max_steps=4)
    w0 = o.w.copy()
    o.train(np.tile(rows[0], (4, 1)), 1)
    params = unpack(w0)
    tl, _ = torch_loss(params, ds.x[:MAXB], ds.y[:MAXB])
    tl.backward()
    g64 = grad_vector(params, w0)
    for s, (loss, w, m) in enumerate(got):
        lr, mu, wd, _ = rows[s]
        assert abs(loss - o.loss[0]) <= 2e-6 * abs(o.loss[0]), (s, loss, o.loss[0])
        check_update(m, w0, wd, g64, off, s)
        # the update is the fused K5 rule on that m, bit for bit: w1 = fma(-lr, m1, w0)
        w_expect = (w0.astype(np.float64) - np.float64(lr) * m.astype(np.float64)).astype(np.float32)
        assert np.max(np.abs(w - w_expect) / np.maximum(np.abs(w_expect), 1e-30)) <= 1.2e-7, s
    # grouping invariance inside the 64-slot launch: equal hp rows give bitwise equal states
    assert all(np.array_equal(got[s][2], got[s + 36][2]) for s in range(SLOTS - 36) if (rows[s] == rows[s + 36]).all())


def test_headline_trajectory_20_steps(ds):
    """(ii) 20 bs-128 steps of 64 grouped slots with lr / momentum switches mid-run; 4 slots of
    different regimes compared with the oracle."""
    n = 20
    base = c2_rows(SLOTS)
    tables = []
    for s in range(SLOTS):
        t = np.tile(base[s], (n + 1, 1))
        t[10:, 0] *= 0.1 if s % 2 == 0 else 1.0    # lr step-decay at 10
        if s % 3 == 1:
            t[5:, 1] = 0.9                         # momentum switch at 5
        tables.append(t)
    pick = [0, 5, 22, 47]
    with cnn_exec() as e:
        for s in range(SLOTS):
            e.slot_init(s)
            e.hp_upload(s, 0, tables[s])
        e.train(list(range(SLOTS)), n)
        got = {s: (e.losses(s, 0, n), e.slot_read(s)[0], e.eval([s])[0]) for s in pick}
    for s in pick:
        o = ol.CnnSlot(ds, max_steps=n + 1)
        o.train(tables[s], n)
        loss, w, (vl, va) = got[s]
        assert np.max(np.abs(loss - o.loss[:n]) / np.abs(o.loss[:n])) <= 1e-4, s
        assert rel(w, o.w) <= 1e-3, (s, rel(w, o.w))
        ovl, ova = o.eval()
        assert abs(vl - ovl) <= 1e-4 * abs(ovl) and abs(va - ova) <= 2 / N_VAL, s


def gaussian_cnn_dataset(seed=7):
    rng = np.random.default_rng(seed)
    d = ol.CnnDataset.__new__(ol.CnnDataset)
    d.n_train = 4096
    d.x = rng.standard_normal((4096 + 64, ol.CNN_SAMPLE), dtype=np.float32)
    d.x.reshape(-1, 1024, 4)[:, :, 3] = 0.0
    d.x[4096:] = d.x[:64]
    d.y = rng.integers(0, 10, 4096 + 64).astype(np.int32)
    d.y[4096:] = d.y[:64]
    d.vx = rng.standard_normal((256, ol.CNN_SAMPLE), dtype=np.float32)
    d.vx.reshape(-1, 1024, 4)[:, :, 3] = 0.0
    d.vy = rng.integers(0, 10, 256).astype(np.int32)
    return d


def test_uploaded_gaussian_data_cnn_tc():
    """(iv) N(0,1) inputs (not exact in tf32) uploaded through smx_dataset_upload, CNN TC mode."""
    d = gaussian_cnn_dataset()
    hp = np.tile(np.float32([1.0, 0.0, 0.0, 64]), (4, 1))
    _, _, off = ol.cnn_layout()
    with ex.Executor(n_slots=2, n_ckpts=1, gemm_mode=ex.GEMM_TC, max_steps=4, max_batch=64, n_train=4096, n_val=256,
                     model=ex.MODEL_CNN) as e:
        e.dataset_upload(d.x, d.y, d.vx, d.vy)
        assert e.dataset_digest() == d.digest()
        e.slot_init(0)
        e.hp_upload(0, 0, hp)
        e.train([0], 1)
        _, m = e.slot_read(0)
        loss = e.losses(0, 0, 1)[0]
    o = ol.CnnSlot(d, max_steps=4)
    w0 = o.w.copy()
    o.train(hp, 1)
    assert abs(loss - o.loss[0]) <= 2e-6 * abs(o.loss[0]), (loss, o.loss[0])
    params = unpack(w0)
    tl, _ = torch_loss(params, d.x[:64], d.y[:64])
    tl.backward()
    check_update(m, w0, 0.0, grad_vector(params, w0), off, "gauss")


def test_uploaded_gaussian_data_mlp_tc():
    """(iv) MLP TC mode: the layer-1 forward and weight gradient read the data operand; with
    non-tf32-exact data they must not take the single-MMA data path."""
    rng = np.random.default_rng(11)
    d = ol.Dataset.__new__(ol.Dataset)
    d.n_train = ol.N_TRAIN
    d.x = rng.standard_normal((ol.N_TRAIN + ol.MAX_BATCH, ol.D0), dtype=np.float32)
    d.x[ol.N_TRAIN:] = d.x[:ol.MAX_BATCH]
    d.y = rng.integers(0, 10, ol.N_TRAIN + ol.MAX_BATCH).astype(np.int32)
    d.y[ol.N_TRAIN:] = d.y[:ol.MAX_BATCH]
    d.vx = rng.standard_normal((ol.N_VAL, ol.D0), dtype=np.float32)
    d.vy = rng.integers(0, 10, ol.N_VAL).astype(np.int32)
    with ex.Executor(n_slots=4, n_ckpts=1, gemm_mode=ex.GEMM_TC, max_steps=32) as e:
        e.dataset_upload(d.x, d.y, d.vx, d.vy)
        for bs in (128, 256):
            hp = np.tile(np.float32([0.1, 0.9, 1e-4, bs]), (4, 1))
            e.slot_init(0)
            e.hp_upload(0, 0, hp)
            e.train([0], 1)
            w, m = e.slot_read(0)
            loss = e.losses(0, 0, 1)[0]
            o = ol.Slot()
            o.train(hp, 1, ds=d)
            assert abs(loss - o.loss[0]) <= 2e-6 * abs(o.loss[0]), (bs, loss, o.loss[0])
            assert rel(m, o.m) <= 2e-5, (bs, rel(m, o.m))
        # eval on the uploaded validation set
        vl, va = e.eval([0])[0]
        ovl, ova = o.eval(ds=d)
        assert abs(vl - ovl) <= 1e-5 * abs(ovl) and abs(va - ova) <= 2 / ol.N_VAL


def c2_mini_spec(T=60):
    """The C2 grid (64 trials: 8 lr step-decays x 8 momentum sequences, bs 128, wd 5e-4) with
    T = 1200 scaled to 60 steps: every milestone / switch step scaled by 1/20."""
    import json
    from pathlib import Path

    spec = json.loads((Path(__file__).resolve().parent.parent / "paper_2006_11972_b200" / "studies" /
                       "c2_grid.json").read_text())
    scale = T / spec["max_steps"]
    spec["name"], spec["max_steps"], spec["eval_interval"] = "c2_mini", T, T // 3
    for fns in spec["space"].values():
        for f in fns:
            if "milestones" in f:
                f["milestones"] = [int(m * scale) for m in f["milestones"]]
    return json.dumps(spec)


def test_c2_mini_engine_tc_vs_cpu_reference_executor():
    """(iii) a truncated C2 study (64 trials, T = 60) through host.Engine in tensor-core mode vs
    the CPU reference executor (oracle/cpu_executor.py: the reference-built plan executed by the
    fp32 oracle): every trial's eval metrics within tolerance; STAGE == TRIAL bitwise in TC mode."""
    import sys
    from pathlib import Path

    from paper_2006_11972_b200 import host

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    import cpu_executor as cx

    spec = c2_mini_spec()
    opts = dict(slots_per_gpu=64, max_batch=MAXB, n_train=N_TRAIN, n_val=N_VAL, gemm_mode=ex.GEMM_TC)
    e = host.Engine.for_study(spec, **opts)
    e.submit_study(spec)
    e.run()
    st = e.stats()
    info = cx.expand_study(spec)
    plan = cx.reference_plan(info["key"], info["trials"])
    unique = sum(n["hi"] - n["start"] for n in plan["node_values"])
    assert st["stage_steps"] == unique and st["trial_steps"] == 64 * 60
    assert st["locksteps"] == 60  # acceptance 8: the critical path
    hist = e.histories()
    # TRIAL mode (every trial unmerged) records bitwise the same metrics
    et = host.Engine.for_study(spec, trial_mode=True, **opts)
    et.submit_study(spec)
    et.run()
    assert et.histories() == hist
    # the CPU reference executor on the reference's plan
    model = cx.Model("cnn", cx.oracle_lib(), n_train=N_TRAIN, max_batch=MAXB, n_val=N_VAL)
    res = cx.run_plan(plan, model, eval_interval=info["eval_interval"])
    assert res["complete"] and res["executed"] == unique
    cpu = cx.trial_histories(plan, res["metrics"])
    worst_l = worst_a = 0.0
    for (study, trial), h in hist.items():
        ref = cpu[(study, trial)]
        assert [s for s, _, _ in h] == sorted(ref), (trial, h, sorted(ref))
        for s, vl, va in h:
            worst_l = max(worst_l, abs(vl - ref[s]["val_loss"]) / abs(ref[s]["val_loss"]))
            worst_a = max(worst_a, abs(va - ref[s]["val_acc"]))
    # 60 SGD steps at lr up to 0.1 / mu 0.9 amplify the 3xTF32 ~1e-6 per-step differences
    # (DESIGN.md §3.6): bound 1e-3 relative on val_loss, 3 of 256 samples on val_acc
    assert worst_l <= 1e-3 and worst_a <= 3 / N_VAL, (worst_l, worst_a)
    print(f"c2_mini: worst val_loss rel {worst_l:.2e}, worst val_acc {worst_a:.4f}")
