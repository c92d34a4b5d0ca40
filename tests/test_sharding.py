"""CPU, world_size 2 over gloo: the multi-GPU reduction the engine relies on.

Each rank simulates the rows r with r % world == rank (the rule
sweep_desc_kernel applies, prologue.cu) into a zero-initialised buffer laid out
like the device row/completion buffers; one all-reduce(SUM) over the raw int64
bits must reproduce the single-process buffers bit for bit (disjoint supports:
x + 0 == x for every 64-bit pattern), so the summary computed afterwards is the
N=1 summary.  The rows themselves come from the CPU oracle here (no GPU in this
container); on the GPU box the same buffers come from the kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2506_19677_b200 as S

MIXES, RPS, CAPS, REPEATS, N_REQ = ["w1", "w3"], [3.0, 12.0], [10, 40], 2, 30


def row_configs():
    out = []
    for m in MIXES:
        for r in RPS:
            for c in CAPS:
                for i in range(REPEATS):
                    out.append((m, r, O.STATIC, c, 42 + i))
            for i in range(REPEATS):
                out.append((m, r, O.SABER, 0, 42 + i))
    return out


def fill(rank, world):
    orc = O.Oracle("restatement")
    cfgs = row_configs()
    rows = np.zeros(len(cfgs), dtype=S.ROW_DTYPE)
    comp = np.zeros((len(cfgs), N_REQ))
    for r, (m, rps, mode, cap, seed) in enumerate(cfgs):
        if r % world != rank:
            continue
        c = O.make_config(mix=m, rps=rps, n=N_REQ, seed=seed, mode=mode, cap=cap)
        res = orc.run(c, records=True)
        o = res.out
        rows[r]["goodput"], rows[r]["ratio_mean"] = o.goodput, o.ratio_mean
        rows[r]["ratio_std"], rows[r]["cv"] = o.ratio_std, o.cv
        rows[r]["n"], rows[r]["completed"], rows[r]["met"] = N_REQ, o.completed, o.met
        rows[r]["decisions"], rows[r]["decision_hash"] = o.decisions, o.decision_hash
        rows[r]["n_kind"] = list(o.n_kind)
        comp[r] = [x.completion_time for x in res.records]
    return rows, comp


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows, comp = fill(rank, world)
    t_rows = torch.from_numpy(rows.view(np.int64).copy())
    t_comp = torch.from_numpy(comp.view(np.int64).copy())
    dist.all_reduce(t_rows)
    dist.all_reduce(t_comp)
    if rank == 0:
        q.put((t_rows.numpy().tobytes(), t_comp.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_disjoint_shards_allreduce_to_the_unsharded_rows(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got_rows, got_comp = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows1, comp1 = fill(0, 1)
    assert got_rows == rows1.view(np.int64).tobytes()
    assert got_comp == comp1.view(np.int64).tobytes()
    # NaN completion times (never completed) survive the integer sum bit-exactly
    assert np.isnan(np.frombuffer(got_comp, dtype=np.float64)).sum() == np.isnan(comp1).sum()
