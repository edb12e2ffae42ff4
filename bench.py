#!/usr/bin/env python
"""Benchmark: trial-equivalent train steps/sec (TES) of a merged HPO study on B200.

A bench "step" is one complete study run through the engine (plan insert -> stage trees ->
critical-path schedule -> grouped GPU training / SAVE / LOAD / EVAL -> metrics recorded), STAGE
mode.  TES = sum over trials of their steps / seconds.

Workloads (`--workload`, default c2 = BASELINE.json configs[1]): c2 the CNN grid (64 trials x
1200 steps, one replica study per rank, weak scaling); c3 N studies over the C3 space merged and
root-partitioned over N ranks (weak); c4_sha / c4_asha tuned C4 studies (replicas); c5 four
studies over one space merged and partitioned (strong).  No collective on the data path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--gemm exact|tc]
                    [--workload c2|c3|c4_sha|c4_asha|c5] [--no-cpu] [--no-trial]

Prints ONE JSON line on rank 0 (contract in the task statement / DESIGN.md §6).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

PEAKS = ROOT / "MEASURED_PEAKS.json"
# DRAM bytes (read + write) per launch of each candidate roofline kernel (64 groups at bs 128,
# max_batch 128) from one `ncu --set full` capture of a 64-slot lockstep
# (profiles/r02/ncu_convs_v17.txt, profiles/debug/r2s3_ncu_all.sh)
TRAFFIC: dict = {
    "K1_conv2_fwd": 1_084_483_000 + 506_878_000,
    "K3_conv2_wgrad": 1_613_938_000 + 70_397_000,
    "K2_conv2_dgrad": 587_761_000 + 1_019_161_000,
    "K2_conv3_dgrad": 364_734_000 + 491_350_000,
    "K1_conv3_fwd": 575_465_000 + 29_468_000,
    "K3_conv3_wgrad": 851_218_000 + 69_658_000,
    "K1_conv1_fwd": 12_789_000 + 1_047_297_000,
    "K3_conv1_wgrad": 1_084_710_000 + 9_852_000,
}
# what each candidate is (tensor-core mode, per launch = 64 groups at bs 128)
KERNEL_DESC: dict = {
    "K1_conv2_fwd": "conv_ws_kernel<Fwd<2>> (conv2 forward implicit GEMM, 64 groups x M 32768 x N 64 x K 288)",
    "K3_conv2_wgrad": "wgrad2_at_kernel (conv2 weight gradient, all 9 taps per persistent CTA, 64 groups x M 289 "
                      "x N 64 x K 32768 in 16 splits)",
    "K2_conv2_dgrad": "conv_ws_kernel<Dgrad<2>> (conv2 input gradient, sub-pixel GEMM, 64 groups x M 8192 x N 128 "
                      "x K 256, 9 of 16 class x neighbour blocks issued)",
    "K2_conv3_dgrad": "conv_ws_kernel<Dgrad<3>> (conv3 input gradient, sub-pixel GEMM, 64 groups x M 2048 x N 2x128 "
                      "x K 256/512)",
    "K1_conv3_fwd": "conv_ws_kernel<Fwd<3>> (conv3 forward implicit GEMM, 64 groups x M 8192 x N 128 x K 576)",
    "K3_conv3_wgrad": "conv_ws_kernel<Wgrad<3>> (conv3 weight gradient, 64 groups x M 577 x N 128 x K 8192 in 4 "
                      "splits; the split reduction with the fused SGD update is a separate kernel)",
}
METRIC = "trial-equivalent train steps/sec per study"
UNIT = "trial-steps/s"


def peaks() -> dict:
    if PEAKS.exists():
        d = json.loads(PEAKS.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback"}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(int(r[0]) for r in self.rows if r[0].isdigit())
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": int(self.rows[0][1]) if self.rows[0][1].isdigit() else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# SMX_BENCH_SHARED_GPU=1: exercise the N > 1 path (rank placement, barriers, max-over-ranks
# timing) with every rank on one GPU and gloo reductions -- a test of the code path, not a number
SHARED_GPU = os.environ.get("SMX_BENCH_SHARED_GPU") == "1"


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if SHARED_GPU:  # test mode: all ranks on the box's GPU(s), gloo for the timing reductions
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def reduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARED_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARED_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


WORKLOADS = {
    # name: (study spec, tuned?, description, slots per GPU, max batch)
    "c2": ("c2_grid", False, "C2 grid (8 lr step-decays x 8 momentum sequences = 64 trials x 1200 steps, bs 128), "
                             "CNN 3x32x32 conv 32/64/128 + GAP + FC, {n} replica stud{ies} (one per rank)", 64, 128),
    "c3": ("c3_random", False, "C3 space x {n} studies (256 random trials x 2000 steps each, seeds 0..{n1}), "
                               "MLP 784-256-256-10, merged plan, root subtrees partitioned over ranks", 128, 256),
    "c4_sha": ("c4_sha", True, "C4 SHA (eta 4, rungs 150/600/1200 steps, 448-trial grid), MLP 784-256-256-10, "
                               "one study per rank (replicas)", 128, 256),
    "c4_asha": ("c4_asha", True, "C4 ASHA (eta 4, rungs 150/600/1200 steps, 448-trial grid, 128 in flight), "
                                 "MLP 784-256-256-10, one study per rank (replicas)", 128, 256),
    "c5": ("c5_space", False, "C5 multi-study merge: 4 studies (256 random trials x 2000 steps each, sampler seeds "
                              "0..3) over one space, one plan (732 leaves, q = 1.868), MLP 784-256-256-10, root "
                              "subtrees partitioned over {n} rank(s)", 128, 256),
}
STRONG = {"c5"}  # fixed total work (4 studies) split over the ranks
DEFAULT_WORKLOAD = "c2"  # BASELINE.json configs[1]: the 1-GPU CNN grid search


def workload(name: str, n_studies: int):
    """Study specs of a workload; sampler seeds 0..n-1 for the partitioned (untuned) ones."""
    from paper_2006_11972_b200 import host

    spec_name, tuned, desc = WORKLOADS[name][:3]
    base = json.loads(host.study_spec(spec_name))
    desc = desc.format(n=n_studies, n1=n_studies - 1, ies="y" if n_studies == 1 else "ies")
    if tuned:
        return [json.dumps(base)], True, desc
    if base.get("sampler", {}).get("kind") != "random":  # grid: identical replica per rank
        return [json.dumps(base)], False, desc
    specs = []
    for s in range(4 if name in STRONG else n_studies):
        sp = dict(base)
        sp["sampler"] = {**base["sampler"], "seed": s}
        specs.append(json.dumps(sp))
    return specs, False, desc


def cuda_time(fn, world):
    """Run fn between device-synchronised CUDA events on torch's stream; max over ranks."""
    import torch

    barrier(world)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    barrier(world)
    return reduce_max(a.elapsed_time(b) / 1e3, world), out


def _spec_text(name: str) -> str:
    return (ROOT / "paper_2006_11972_b200" / "studies" / f"{WORKLOADS[name][0]}.json").read_text()


class CpuReference:
    """The reference's CPU path for a workload (oracle/cpu_executor.py): the merged plan built by
    the compiled reference (oracle/_ref: SearchPlan::insert_trial / value_at), executed with the
    stage executor's resume / fork / eval semantics by the CPU oracle trainer (liboracle_v4.so,
    AVX-512, when the host has it) on every host core.  Imports nothing from
    paper_2006_11972_b200.  A sample runs the plan from scratch for a bounded wall budget; TES is
    the study's trial-steps x (executed / unique stage-steps) / wall seconds."""

    def __init__(self, workload_name: str, max_batch: int):
        sys.path.insert(0, str(ROOT / "oracle"))
        import cpu_executor as cx

        self.cx = cx
        spec = json.loads(_spec_text(workload_name))
        if spec.get("tuner"):
            raise ValueError("the CPU reference executes untuned plans only")
        self.info = cx.expand_study(spec)
        self.plan = cx.reference_plan(self.info["key"], self.info["trials"])
        self.lib = cx.oracle_lib()
        self.model = cx.Model(self.info["key"]["model"], self.lib, n_train=65536, max_batch=max_batch, n_val=4096)
        self.cores = os.cpu_count() or 1
        self.unique = sum(n["hi"] - n["start"] for n in self.plan["node_values"])
        self.trial_steps = cx.total_trial_steps(self.plan)

    def sample(self, budget_s: float) -> dict:
        r = self.cx.run_plan(self.plan, self.model, eval_interval=self.info["eval_interval"], threads=self.cores,
                             budget_s=budget_s)
        frac = r["executed"] / self.unique
        tes = self.trial_steps * frac / r["wall_s"]
        return {"value": tes, "unit": UNIT, "cores": self.cores, "kind": "port",
                "same_config": True, "fraction_executed": frac,
                "sample": f"{self.info['name']}: the reference-built plan ({len(self.plan['node_values'])} nodes, "
                          f"{self.unique} unique stage-steps, {self.trial_steps} trial-steps) executed from scratch "
                          f"for a {budget_s:.0f} s wall budget: {r['executed']} stage-steps + "
                          f"{len(r['metrics'])} evals in {r['wall_s']:.1f} s ({frac * 100:.2f} % of the study; "
                          f"{r['executed'] / r['wall_s']:.1f} stage-steps/s) on {self.cores} threads, "
                          f"oracle {self.lib.isa}; TES = trial-steps x fraction / wall",
                "executed_stage_steps": r["executed"], "wall_s": r["wall_s"]}

    @staticmethod
    def libraries() -> list:
        maps = Path("/proc/self/maps")
        if not maps.exists():
            return []
        return sorted({l.split()[-1] for l in maps.read_text().splitlines() if l.endswith(".so") and str(ROOT) in l})


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path (CpuReference), rank 0
    only (other ranks exit 0 without work); nothing of paper_2006_11972_b200 is imported."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    desc = WORKLOADS[args.workload][2].format(n=1, n1=0, ies="y")
    ref = CpuReference(args.workload, WORKLOADS[args.workload][4])
    budget = max(3.0, min(20.0, 150.0 / (args.warmup + args.steps)))
    vals, cb = [], None
    for i in range(args.warmup + args.steps):
        cb = ref.sample(budget)
        if i >= args.warmup:
            vals.append(cb["value"])
    v = float(np.mean(vals))
    libs = CpuReference.libraries()
    assert not any("paper_2006_11972_b200" in l for l in libs), libs
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                      "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                      "config": {"workload": desc, "flush": "n/a (CPU)", "same_config": True},
                      "cpu_baseline": {**cb, "value": v}, "native_so_loaded": libs,
                      "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gemm", default=os.environ.get("SMX_BENCH_GEMM", "tc"), choices=["exact", "tc"])
    ap.add_argument("--slots", type=int, default=0, help="slots per GPU (0: the workload's default)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--no-trial", action="store_true", help="skip the TRIAL-mode (unmerged) comparison run")
    args = ap.parse_args()
    if not args.slots:
        args.slots = WORKLOADS[args.workload][3]
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_init()

    import torch

    from paper_2006_11972_b200 import executor as ex
    from paper_2006_11972_b200 import host

    torch.cuda.set_device(local)
    specs, tuned, desc = workload(args.workload, world)
    info = host.expand_study(specs[0])
    gemm_mode = ex.GEMM_TC if args.gemm == "tc" else ex.GEMM_EXACT
    # random-sampled studies differ per rank and are merged + root-partitioned; tuned studies and
    # grids run one replica per rank
    partitioned = not tuned and world > 1 and (len(specs) == world or args.workload in STRONG)
    part = {"rank": rank, "world": world} if partitioned else {}
    cnn = info["key"]["model"] == "cnn"
    max_batch = WORKLOADS[args.workload][4]
    eng = host.Engine.for_study(specs[0], devices=[local], slots_per_gpu=args.slots, ckpts_per_gpu=1024,
                                gemm_mode=gemm_mode, max_steps=2048, max_batch=max_batch, **part)

    def submit_and_run(e):
        if tuned:
            e.run_tuned(specs)
        else:
            for s, sp in enumerate(specs):
                e.submit_study(sp, s)
            e.run()

    def one_study():
        eng.reset()
        submit_and_run(eng)
        return eng.stats()

    for _ in range(args.warmup):
        one_study()
    with Clocks(local) as clk:
        t, st = cuda_time(lambda: [one_study() for _ in range(args.steps)][-1], world)
    trial_steps = reduce_sum(st["trial_steps"], world)  # the study's trials, split over ranks
    stage_steps = reduce_sum(st["stage_steps"], world)
    value = trial_steps * args.steps / t

    # ---- e2e: the same study through the public Engine API with the dataset coming from
    # pinned host memory every step (H2D inside the timed region) and metrics read back (D2H).
    # The host copy is staged once, outside the timed region, by reading the context's dataset
    # back (smx_dataset_read) into page-locked buffers.
    import ctypes

    lib = ex.load_library()
    d_in = 32 * 32 * 4 if cnn else 784
    rows = 65536 + max_batch
    shapes = [((rows, d_in), np.float32), ((rows,), np.int32), ((4096, d_in), np.float32), ((4096,), np.int32)]
    pinned, host_arrays = [], []
    for shape, dt in shapes:
        nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
        p = ctypes.c_void_p()
        assert lib.smx_host_alloc(nbytes, ctypes.byref(p)) == 0
        host_arrays.append(np.ctypeslib.as_array((ctypes.c_byte * nbytes).from_address(p.value)).view(dt).reshape(shape))
        pinned.append(p)
    ctx0 = ctypes.c_void_p(eng.context_ptrs()[0])
    ex._check(lib.smx_dataset_read(ctx0, *[a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)) if a.dtype == np.float32
                                           else a.ctypes.data for a in host_arrays]))
    digest0 = eng.dataset_digest()

    def one_e2e():
        eng.reset()
        eng.upload_dataset(*host_arrays)
        submit_and_run(eng)
        return eng.stats()

    one_e2e()
    te, st_e = cuda_time(lambda: [one_e2e() for _ in range(args.steps)][-1], world)
    e2e_value = reduce_sum(st_e["trial_steps"], world) * args.steps / te
    assert eng.dataset_digest() == digest0, "e2e upload changed the dataset"
    del host_arrays
    for p in pinned:
        lib.smx_host_free(p)

    # ---- GPU-second savings: the same studies unmerged (TRIAL mode: every trial on its own
    # path) on the same executor, device-timed once after one warm-up run
    savings = None
    if not args.no_trial:
        teng = host.Engine.for_study(specs[0], devices=[local], slots_per_gpu=args.slots, ckpts_per_gpu=1024,
                                     gemm_mode=gemm_mode, max_steps=2048, max_batch=max_batch, trial_mode=True,
                                     **part)

        def one_trial():
            teng.reset()
            submit_and_run(teng)
            return teng.stats()

        one_trial()
        tt, st_t = cuda_time(one_trial, world)
        savings = {"stage_gpu_s": t / args.steps, "trial_gpu_s": tt, "ratio": tt / (t / args.steps),
                   "trial_mode_stage_steps": reduce_sum(st_t["stage_steps"], world),
                   "trial_mode_trial_steps": reduce_sum(st_t["trial_steps"], world),
                   "executed_merge_rate": trial_steps / stage_steps,
                   "note": "GPU-busy seconds TRIAL / STAGE on the same executor (SPEC.md:396-398: tracks the "
                           "executed merge rate when per-step cost is uniform)"}
        del teng

    # ---- per-kernel roofline: standalone CUDA-event timing of the dominant kernels on a fresh
    # 64-slot context of the same GPU (bs 128, the study's typical active set)
    pk = peaks()
    n_k = 64
    kx = ex.Executor(n_slots=n_k, n_ckpts=16, device=local, max_steps=64, gemm_mode=gemm_mode, max_batch=max_batch,
                     model=ex.MODEL_CNN if cnn else ex.MODEL_MLP)
    for s_ in range(n_k):
        kx.slot_init(s_)
        kx.hp_upload(s_, 0, np.tile(np.float32([0.05, 0.9, 1e-4, 128]), (64, 1)))
    kx.train(list(range(n_k)), 1)  # produce activations / gradients once
    kx.sync()
    # CNN: 2 / 3 = conv2 forward / weight gradient, 4 / 5 = conv2 / conv3 input gradient, 6 = conv3
    # forward, 7 = conv3 weight gradient (+ its split reduction); MLP: 2 / 3 only
    # 8 / 9 = conv1 weight gradient (+ reduction) / forward, both HBM-bound tensor-core kernels
    ms = {kind: kx.bench_kernel(kind, n_k, 30) for kind in ((2, 3, 4, 5, 6, 7, 8, 9) if cnn else (2, 3))}
    # HBM-bound kernels on a working set > 3x the 126 MB L2 (many small slots / checkpoints)
    n_h = int(np.ceil(3 * 126e6 / (20 * kx.p_algo * 1.0) / 16)) * 16
    kh = ex.Executor(n_slots=n_h, n_ckpts=n_h, device=local, max_steps=8, gemm_mode=gemm_mode, max_batch=8,
                     n_train=4096, n_val=256, model=ex.MODEL_CNN if cnn else ex.MODEL_MLP)
    for s_ in range(n_h):
        kh.slot_init(s_)
        kh.hp_upload(s_, 0, np.tile(np.float32([0.05, 0.9, 1e-4, 8]), (8, 1)))
    kh.sync()
    ms[0] = kh.bench_kernel(0, n_h, 20)
    ms[1] = kh.bench_kernel(1, n_h, 20)
    kh.close()
    P = kx.p_algo
    kx.close()
    upd_bytes, fork_bytes = 20 * P * n_h, 16 * P * n_h
    if cnn:  # conv2: M = 128 x 16 x 16 output pixels, N = 64, K = 9 x 32 (forward; the weight
        # gradient is the same product count with M and K exchanged)
        gemm_flops = 2 * 128 * 256 * 288 * 64 * n_k
    else:  # layer 1: 128 x 256 x 784 (both kinds)
        gemm_flops = 2 * 128 * 256 * 784 * n_k
    tc_peak = pk["bf16_tflops"]

    def hbm(name, b, t, **kw):
        a = b / (t * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": a, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": a / pk["hbm_gbs"],
                "bytes_per_launch": b, "ms_per_launch": t, "peak_src": pk["src"], **kw}

    def tensor(name, f, t):
        a = f / (t * 1e-3) / 1e12
        return {"bound": "tensor", "achieved": a, "peak": tc_peak, "unit": "TFLOP/s", "frac": a / tc_peak,
                "flops_per_launch": f, "ms_per_launch": t, "peak_src": pk["src"] + " bf16 dense",
                "note": "fp32-equivalent flops; 3xTF32 issues 3 kind::tf32 MMAs (tf32 = bf16/2) per product, so "
                        "the mode's own ceiling is bf16/6 = %.0f TFLOP/s" % (tc_peak / 6)}

    if cnn:
        kernels = {
            "K1_conv2_fwd": tensor("fwd", gemm_flops, ms[2]),
            "K3_conv2_wgrad": tensor("wgrad", gemm_flops, ms[3]),
            # every conv2 / conv3 implicit GEMM has the same algorithmic product count per sample
            # (2 x 256 x 64 x 288 = 2 x 64 x 128 x 576); the input gradients issue 16/9 of it
            "K2_conv2_dgrad": tensor("dgrad2", gemm_flops, ms[4]),
            "K2_conv3_dgrad": tensor("dgrad3", gemm_flops, ms[5]),
            "K1_conv3_fwd": tensor("fwd3", gemm_flops, ms[6]),
            "K3_conv3_wgrad": tensor("wgrad3", gemm_flops, ms[7]),
            # conv1 (tensor cores, HBM-bound): the forward writes a1 (128 x 1024 x 32 fp32 per slot)
            # and reads the images (128 x 4096 fp32); the weight gradient reads dA1 and the images
            "K1_conv1_fwd": hbm("fwd1", n_k * 128 * (1024 * 32 + 4096) * 4, ms[9], traffic=TRAFFIC["K1_conv1_fwd"]),
            "K3_conv1_wgrad": hbm("wgrad1", n_k * 128 * (1024 * 32 + 4096) * 4, ms[8], traffic=TRAFFIC["K3_conv1_wgrad"]),
            "K5_update": hbm("upd", upd_bytes, ms[0], slots=n_h),
            "K6_fork": hbm("fork", fork_bytes, ms[1], checkpoints=n_h),
        }
        # the roofline kernel is the dominant one: the longest of the six implicit GEMMs (each has the
        # same algorithmic product count per launch), i.e. the largest share of the lockstep
        dom = max(KERNEL_DESC, key=lambda k: kernels[k]["ms_per_launch"]) if gemm_mode == ex.GEMM_TC else "K3_conv2_wgrad"
        roofline = dict(kernels[dom])
        roofline["kernel"] = KERNEL_DESC[dom] if gemm_mode == ex.GEMM_TC else "conv_wgrad_simt<2>"
        roofline["traffic"] = TRAFFIC.get(dom) if gemm_mode == ex.GEMM_TC else None
    else:
        kernels = {
            "K1_fwd1_gemm": tensor("fwd1", gemm_flops, ms[2]),
            "K3_wgrad1_gemm": tensor("wgrad1", gemm_flops, ms[3]),
            "K5_update": hbm("upd", upd_bytes, ms[0], slots=n_h),
            "K6_fork": hbm("fork", fork_bytes, ms[1], checkpoints=n_h),
        }
        roofline = dict(kernels["K1_fwd1_gemm"])
        roofline["kernel"] = "conv_ws_kernel<DenseOp<0,0,BiasRelu,exact A>> (MLP layer-1 forward, 64 groups x 128x256x784)"
        roofline["traffic"] = None

    # ---- K7: checkpoint fork to another GPU (smx_ckpt_peer_copy, NVLink P2P); on a 1-GPU box the
    # same call between two contexts of the one device (a device-local copy), labelled as such
    k7 = None
    if rank == 0 and world == 1:
        ndev = torch.cuda.device_count()
        src_dev, dst_dev = local, (local + 1) % ndev if ndev > 1 else local
        mk = dict(max_steps=8, max_batch=8, n_train=4096, n_val=256, gemm_mode=gemm_mode,
                  model=ex.MODEL_CNN if cnn else ex.MODEL_MLP)
        n7 = 32
        src = ex.Executor(n_slots=1, n_ckpts=n7, device=src_dev, **mk)
        dst = ex.Executor(n_slots=1, n_ckpts=n7, device=dst_dev, **mk)
        src.slot_init(0)
        for i in range(n7):
            src.slot_save(0, i)
        for i in range(n7):
            dst.ckpt_peer_copy(i, src, i)
        # the engine's call (one checkpoint, event-ordered against both contexts), CUDA events
        dst.set_timing(True)
        dst.reset_stats()
        for _ in range(3):
            for i in range(n7):
                dst.ckpt_peer_copy(i, src, i)
        kst = dst.stats()
        ms1 = kst["fork_ms"] / kst["fork_launches"]
        dst.set_timing(False)
        # the kernel's bandwidth: 16 checkpoints per launch, 20 launches between events
        ms7 = dst.bench_peer_copy(src, 16, 20)
        b7 = 8 * src.p_alloc + 16  # w | m + step / offset, one direction
        link = src_dev != dst_dev
        a7 = b7 / (ms7 * 1e-3) / 1e9
        # same device: the copy reads and writes HBM (2 x the bytes against the copy bandwidth)
        peak7 = 900.0 if link else pk["hbm_gbs"] / 2
        k7 = {"bound": "nvlink" if link else "hbm (same device: no peer on this box)", "achieved": a7,
              "peak": peak7, "unit": "GB/s", "frac": a7 / peak7, "bytes_per_copy": b7, "ms_per_copy": ms7,
              "ms_per_single_call": ms1, "devices": [src_dev, dst_dev],
              "note": "16 checkpoints per launch; ms_per_single_call = one engine LOAD (latency-bound at 0.76 MB)"}
        src.close()
        dst.close()

    cpu = None
    if rank == 0 and not args.no_cpu and not tuned and world == 1:
        cpu = CpuReference(args.workload, max_batch).sample(20.0)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.workload in STRONG else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": desc,
                       "gemm": args.gemm, "slots_per_gpu": args.slots, "trials": len(info["trials"]) * len(specs),
                       "trial_steps": trial_steps, "unique_stage_steps": stage_steps,
                       "executed_merge_rate": trial_steps / stage_steps,
                       "flush": ("inputs > L2: per-slot activations 60 MB x 64 slots + 1.07 GB dataset" if cnn else
                                 "inputs > L2: per-slot state 2.2 MB x 128 slots + 206 MB dataset")},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": st_e["h2d_bytes"], "d2h_bytes_per_step": st_e["d2h_bytes"]},
            "gpu_launches": st["kernel_launches"] * args.steps,
            "roofline": roofline,
            "kernels": {**kernels, **({"K7_peer_fork": k7} if k7 else {})},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "engine_stats": st,
            "gpu_seconds_savings": savings,
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
