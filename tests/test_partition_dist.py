"""Multi-GPU placement without GPUs: two gloo ranks each build the C3 plan, compute
the root-subtree LPT partition the engine uses (stagemerge::assign_roots) and check, through
collectives, that every rank derived the identical map, that ranks own disjoint subtrees covering
the whole plan, and that the load is balanced.  No collective is needed on the data path; this
test only uses gloo to compare the ranks' independent decisions."""
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_11972_b200 import host


def plan_cmd(n_studies: int, world: int) -> dict:
    actions, rid = [], 0
    key = None
    for s in range(n_studies):
        spec = json.loads(host.study_spec("c3_random"))
        spec["sampler"]["seed"] = s
        info = host.expand_study(json.dumps(spec))
        key = info["key"]
        for t, cfg in enumerate(info["trials"]):
            actions.append({"kind": "insert", "id": (s << 32) | t, "study": s, "trial": t, "config": cfg})
            rid += 1
    return {"op": "plan", "key": key, "actions": actions, "partition": world}


def _worker(rank, world, port, n_studies, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = host.call(plan_cmd(n_studies, world))
    owner = r["partition"]["owner"]
    mine = sorted(int(k) for k, v in owner.items() if v == rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, {"owner": owner, "mine": mine, "sig": r["signature"],
                                      "work": r["partition"]["work"]})
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n_studies", [1, 2])
def test_two_rank_partition_agrees_and_covers(n_studies):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_studies, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(g["owner"] == gathered[0]["owner"] for g in gathered)  # independent but identical decisions
    assert all(g["sig"] == gathered[0]["sig"] for g in gathered)      # identical plans
    mine = [set(g["mine"]) for g in gathered]
    assert mine[0].isdisjoint(mine[1])
    roots = {int(k) for k in gathered[0]["owner"]}
    assert mine[0] | mine[1] == roots
    work = {int(k): v for k, v in gathered[0]["work"].items()}
    load = [sum(work[r] for r in m) for m in mine]
    assert min(load) > 0 and max(load) / sum(load) < 0.75, load
