"""GPU parity of the stage executor (C ABI) against the CPU oracle.

Exact mode (SMX_GEMM_EXACT) must be bit-identical to oracle/trainer.c: losses, weights,
momentum, data offsets and eval metrics.  Grouping invariance and STAGE == TRIAL equality are
checked bitwise on the GPU itself (plan.cpp:172-179)."""
import numpy as np
import pytest

from oracle_lib import Slot, dataset
from paper_2006_11972_b200 import executor as ex

pytestmark = pytest.mark.gpu


def hp_const(n, lr=0.1, mu=0.9, wd=1e-4, bs=128):
    return np.tile(np.float32([lr, mu, wd, bs]), (n, 1))


@pytest.fixture(scope="module")
def gpu():
    e = ex.Executor(n_slots=8, n_ckpts=8, max_steps=512)
    yield e
    e.close()


def test_dataset_bitwise_equal_to_oracle(gpu):
    assert gpu.dataset_digest() == dataset().digest()


def test_init_bitwise_equal_to_oracle(gpu):
    gpu.slot_init(0)
    w, m = gpu.slot_read(0)
    o = Slot()
    assert np.array_equal(w, o.w) and np.array_equal(m, o.m)
    assert gpu.slot_state(0) == (0, 0)


@pytest.mark.parametrize("graphs", [True, False])
def test_exact_training_bitwise_equal_to_oracle(gpu, graphs):
    hp = hp_const(30)
    hp[:, 0] = np.float32(0.1) * np.float32(0.95) ** np.arange(30, dtype=np.float32)  # per-step lr
    hp[12:, 3] = 96  # ragged batch (not a multiple of 64) from step 12
    gpu.set_graphs(graphs)
    gpu.slot_init(1)
    gpu.hp_upload(1, 0, hp)
    gpu.train([1], 12)
    gpu.train([1], 18)
    w, m = gpu.slot_read(1)
    losses = gpu.losses(1, 0, 30)
    o = Slot()
    o.train(hp, 30)
    assert gpu.slot_state(1) == (30, o.offset.value)
    assert np.array_equal(losses, o.loss[:30])
    assert np.array_equal(w, o.w)
    assert np.array_equal(m, o.m)
    gpu.set_graphs(True)


def test_grouping_invariance(gpu):
    """A slot's trajectory does not depend on which other slots share the launch."""
    hps = [hp_const(10, lr=lr, bs=bs) for lr, bs in [(0.1, 128), (0.05, 64), (0.2, 256), (0.01, 32)]]
    for s, hp in enumerate(hps):
        gpu.slot_init(s)
        gpu.hp_upload(s, 0, hp)
    gpu.train([0, 1, 2, 3], 10)
    together = [gpu.slot_read(s)[0] for s in range(4)]
    for s, hp in enumerate(hps):
        gpu.slot_init(4)
        gpu.hp_upload(4, 0, hp)
        gpu.train([4], 10)
        assert np.array_equal(gpu.slot_read(4)[0], together[s]), s


def test_fork_save_load_and_stage_equals_trial(gpu):
    """Fig. 1 shape: shared prefix of 20 steps, then two children.  Merged execution (train the
    prefix once, SAVE, LOAD into two slots) equals two independent runs bitwise."""
    prefix = hp_const(20, lr=0.1)
    tail_a, tail_b = hp_const(15, lr=0.01), hp_const(15, lr=0.001, bs=64)
    hp_a, hp_b = np.vstack([prefix, tail_a]), np.vstack([prefix, tail_b])
    # STAGE mode
    gpu.slot_init(0)
    gpu.hp_upload(0, 0, prefix)
    gpu.train([0], 20)
    gpu.slot_save(0, 3)
    for s, hp in [(1, hp_a), (2, hp_b)]:
        gpu.slot_load(s, 3)
        gpu.hp_upload(s, 0, hp)
    gpu.train([1, 2], 15)
    stage = [gpu.slot_read(s) for s in (1, 2)] + [gpu.eval([1, 2])]
    # TRIAL mode
    for s, hp in [(5, hp_a), (6, hp_b)]:
        gpu.slot_init(s)
        gpu.hp_upload(s, 0, hp)
        gpu.train([s], 35)
    trial = [gpu.slot_read(s) for s in (5, 6)] + [gpu.eval([5, 6])]
    for (ws, ms), (wt, mt) in zip(stage[:2], trial[:2]):
        assert np.array_equal(ws, wt) and np.array_equal(ms, mt)
    assert np.array_equal(stage[2], trial[2])
    # and the oracle agrees
    o = Slot()
    o.train(hp_b, 35)
    assert np.array_equal(trial[1][0], o.w)
    assert tuple(trial[2][1]) == o.eval()


def test_eval_bitwise_equal_to_oracle(gpu):
    gpu.slot_init(7)
    gpu.hp_upload(7, 0, hp_const(5))
    gpu.train([7], 5)
    o = Slot()
    o.train(hp_const(5), 5)
    got = gpu.eval([7])[0]
    assert tuple(got) == o.eval()


def test_checkpoint_roundtrip_and_integrity(gpu):
    gpu.slot_init(0)
    gpu.slot_save(0, 0)
    w, m, step, off = gpu.ckpt_read(0)
    assert step == 0 and off == 0 and np.array_equal(w, Slot().w)
    gpu.ckpt_free(0)
    with pytest.raises(ex.SmxIntegrityError):
        gpu.slot_load(1, 0)
    with pytest.raises(ex.SmxConfigError):
        gpu.hp_upload(0, 510, hp_const(5))
    with pytest.raises(ex.SmxConfigError):
        gpu.hp_upload(0, 0, hp_const(1, bs=300))
    with pytest.raises(ex.SmxConfigError):
        gpu.train([0, 0], 1)


def test_update_and_fork_kernels_bench(gpu):
    ms_u = gpu.bench_kernel(0, 8, 20)
    ms_f = gpu.bench_kernel(1, 8, 20)
    assert ms_u > 0 and ms_f > 0
