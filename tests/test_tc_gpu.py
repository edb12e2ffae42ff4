"""Tensor-core mode (SMX_GEMM_TC: tcgen05 kind::tf32, 3xTF32) against the CPU fp32 oracle.

Stated tolerance: the 3xTF32 GEMMs reproduce fp32 to ~1e-6 relative per
GEMM.  Over a run, SGD amplifies any 1e-6 difference at a regime-dependent rate (the fp32
oracle itself, with its initial weights perturbed by 1e-6 relative, drifts 1e-5 in a gentle
regime and 6e-2 in an aggressive one), so the multi-step bound is stated against that intrinsic
envelope:
  * first-step loss:                   |rel| <= 2e-6
  * first-step update (m = g + wd w):  rel L2 <= 2e-5
  * 200 steps, lr 0.01 / mu 0.5:       loss max |rel| <= 1e-4, weights rel L2 <= 1e-3
  * 200 steps, lr 0.05 / mu 0.9:       within 3x the oracle's own 1e-6-perturbation drift
STAGE == TRIAL and grouping invariance are bitwise in this mode too (deterministic kernels)."""
import numpy as np
import pytest

from oracle_lib import Slot
from paper_2006_11972_b200 import executor as ex
from paper_2006_11972_b200 import host

pytestmark = pytest.mark.gpu


def hp_const(n, lr=0.1, mu=0.9, wd=1e-4, bs=128):
    return np.tile(np.float32([lr, mu, wd, bs]), (n, 1))


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30))


@pytest.fixture(scope="module")
def tc():
    e = ex.Executor(n_slots=8, n_ckpts=4, max_steps=512, gemm_mode=ex.GEMM_TC)
    yield e
    e.close()


@pytest.mark.parametrize("bs", [128, 256, 96, 32])
def test_first_step_matches_oracle(tc, bs):
    hp = hp_const(1, bs=bs)
    tc.slot_init(0)
    tc.hp_upload(0, 0, hp)
    tc.train([0], 1)
    w, m = tc.slot_read(0)
    o = Slot()
    o.train(hp, 1)
    l_tc, l_or = tc.losses(0, 0, 1)[0], o.loss[0]
    assert abs(l_tc - l_or) / l_or <= 2e-6, (l_tc, l_or)
    assert rel(m, o.m) <= 2e-5, rel(m, o.m)
    assert rel(w, o.w) <= 1e-6


def run_both(tc, slot, hp):
    tc.slot_init(slot)
    tc.hp_upload(slot, 0, hp)
    tc.train([slot], hp.shape[0])
    w, _ = tc.slot_read(slot)
    o = Slot()
    o.train(hp, hp.shape[0])
    lt = tc.losses(slot, 0, hp.shape[0])
    err = np.abs(lt - o.loss[:hp.shape[0]]) / o.loss[:hp.shape[0]]
    return w, lt, o, err


def test_trajectory_gentle_regime(tc):
    hp = hp_const(200, lr=0.01, mu=0.5)
    hp[100:, 3] = 256
    w, _, o, err = run_both(tc, 1, hp)
    print("gentle: max rel loss err", err.max(), "weights rel err", rel(w, o.w))
    assert err.max() <= 1e-4
    assert rel(w, o.w) <= 1e-3
    got, want = tc.eval([1])[0], o.eval()
    assert abs(got[0] - want[0]) / want[0] <= 1e-4


def test_trajectory_aggressive_regime_within_intrinsic_envelope(tc):
    hp = hp_const(200, lr=0.05, mu=0.9)
    hp[100:, 3] = 256
    w, _, o, err = run_both(tc, 2, hp)
    p = Slot()
    rng = np.random.default_rng(0)
    p.w[:] = p.w * (1 + rng.standard_normal(p.w.size).astype(np.float32) * 1e-6)
    p.train(hp, 200)
    env = np.abs(p.loss[:200] - o.loss[:200]) / o.loss[:200]
    print("aggressive: tc", err.max(), rel(w, o.w), "oracle 1e-6 envelope", env.max(), rel(p.w, o.w))
    assert err.max() <= 3 * env.max()
    assert rel(w, o.w) <= 3 * rel(p.w, o.w)


def test_tc_grouping_invariance_and_determinism(tc):
    hps = [hp_const(6, lr=lr, bs=bs) for lr, bs in [(0.1, 128), (0.05, 64), (0.2, 256)]]
    for s, hp in enumerate(hps):
        tc.slot_init(s)
        tc.hp_upload(s, 0, hp)
    tc.train([0, 1, 2], 6)
    together = [tc.slot_read(s)[0] for s in range(3)]
    for s, hp in enumerate(hps):
        tc.slot_init(5)
        tc.hp_upload(5, 0, hp)
        tc.train([5], 6)
        assert np.array_equal(tc.slot_read(5)[0], together[s]), s


def test_tc_engine_stage_equals_trial():
    spec = host.study_spec("c1_fig1")
    runs = []
    for trial_mode in (False, True):
        e = host.Engine.for_study(spec, slots_per_gpu=4, gemm_mode=ex.GEMM_TC, trial_mode=trial_mode)
        e.submit_study(spec)
        e.run()
        runs.append(e.histories())
    assert runs[0] == runs[1]
