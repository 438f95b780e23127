"""World-size-2 host-side tests over gloo on CPU (no GPU): the N > 1 bootstrap
path of bench.py / the engine — NCCL unique-id creation on rank 0 and its
broadcast through torch.distributed, per-rank planning that must agree across
processes (shard ranges tile every bucket, per-rank bytes sum to the closed
form), and the max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import accounting as A
        from paper_2310_06003_b200 import paro
        from paro_synth import llama_param_sizes

        # uid creation on rank 0 and broadcast (bench.py path)
        uid = paro.unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8)
        dist.broadcast(t, 0)
        uid = bytes(t.tolist())
        got = [None] * world
        dist.all_gather_object(got, uid)
        assert len(uid) == 128 and all(g == got[0] for g in got)

        sizes = llama_param_sizes("7B")
        N, M = 8, 4     # plan an 8-rank job from 2 processes (planning is host-only)
        ctx = paro.Context(N, M)
        for code in ("IIG", "NIG", "IGG", "NNN", "III"):
            pl = paro.Plan(ctx, code, sizes, bucket_elems=1 << 26)
            info = pl.info()
            mine = [pl.shard_range("OS", r, b) for r in range(rank, N, world) for b in (0, 50, 100)]
            allr = [None] * world
            dist.all_gather_object(allr, mine)
            flat = sorted(x for part in allr for x in part)
            for b in (0, 50, 100):
                lo, hi = pl.bucket_range(b)
                segs = sorted(x for x in flat if lo <= x[0] < hi)
                if code[2] == "G":
                    assert segs[0][0] == lo and segs[-1][1] == hi
                    assert all(segs[i][1] == segs[i + 1][0] for i in range(len(segs) - 1))
            sent = sum(sum(pl.send_bytes(r)) for r in range(rank, N, world))
            tot = torch.tensor([sent], dtype=torch.int64)
            dist.all_reduce(tot)
            a, b_ = A.step_units_per_rank(code, N, M, info["psi_pad"])
            assert int(tot.item()) == N * 2 * (a + b_)
            pl.close()
        ctx.close()
        # max-over-ranks step time (bench.py)
        ms = torch.tensor([10.0 + rank], dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        assert ms.item() == 10.0 + world - 1
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_bootstrap_and_planning():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
