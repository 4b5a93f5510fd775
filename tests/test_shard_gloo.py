"""Multi-GPU work split exercised on CPU with world_size 2
over gloo: each rank counts only its share of the (task, level-2 chunk) work
units under the cost-balanced rule floor(world * prefix / total); the
all-reduced counts must equal the unsharded counts (and the reference's)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_util as gu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, suite, names, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_py import Oracle
    results = []
    for inst in gu.load(suite):
        if names and inst["name"] not in names:
            continue
        vl, eu, ev, el, ql, qe, batches = gu.instance_arrays(inst)
        o = Oracle(vl, eu, ev, el)
        o.add_query(ql, qe)
        for b in batches:
            pos, neg, _ = o.apply_batch(b, rank=rank, world=world)
            t = torch.tensor([pos[0], neg[0]], dtype=torch.int64)
            dist.all_reduce(t)
            results.append(t.tolist())
    if rank == 0:
        out.put(results)
    dist.barrier()
    dist.destroy_process_group()


def _run(suite, names=None, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, suite, names, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("suite", ["streams", "skewed"])
def test_sharded_counts_sum_to_reference(suite):
    insts = gu.load(suite)
    if suite == "streams":
        insts = insts[-6:]
    names = [i["name"] for i in insts]
    got = _run(suite, names)
    exp = [[e["pos"], e["neg"]] for i in insts for e in i["expect"]]
    assert got == exp


def test_shard_owner_rule_matches_engine_rule():
    """The CPU restatement and the C ABI share the owner rule."""
    import paper_2401_17018_b200 as bd
    costs = [64, 64, 17, 64, 3, 1, 1, 64, 64, 64, 12]
    total = sum(costs)
    for world in (2, 4, 8):
        prefix, expect = 0, []
        for c in costs:
            expect.append(prefix * world // total)
            prefix += c
        assert bd.shard_owners(costs, world) == expect
