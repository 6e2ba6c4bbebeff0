"""bench.py's c5 rank loop on CPU (-m "not gpu"): the fixed global batch split by
dist.shard_range, calls of F frames per rank, per-frame checksums gathered over gloo in
global frame order.  The GPU call is stubbed by the fp64 oracle on tiny frames; the
digest must be the same for world sizes 1, 2 and 3 (frames are independent,
P:561-563)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

BATCH, W, H, Q = 7, 48, 32, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_loop(rank, world):
    import bench
    import oracle
    from paper_2410_11625_b200 import synth

    lo, hi, F, pool, seeds = bench.batch_plan(BATCH, rank, world, frames_per_call=2)
    assert pool * F == hi - lo and len(seeds) == hi - lo

    def call(i):  # oracle stand-in for the denoise call on the i-th chunk of the shard
        outs = []
        for s in seeds[i * F:(i + 1) * F]:
            G, Y = synth.frame(W, H, Q=Q, seed=s)
            outs.append(oracle.denoise(G.numpy(), Y.numpy(), D=8, sigma=10.0, R=3)[0])
        return torch.from_numpy(np.stack(outs))

    return bench.batch_checksums(call, pool, lo, BATCH), (lo, hi)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cs, span = _rank_loop(rank, world)
        q.put((rank, cs, span))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_batch_rank_loop_digest_independent_of_world(world):
    ref, span = _rank_loop(0, 1)
    assert span == (0, BATCH) and ref["frames"] == BATCH and ref["all_finite"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spans = sorted(s for _, _, s in got)
    assert spans[0][0] == 0 and spans[-1][1] == BATCH
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:])), spans  # contiguous, disjoint
    for _, cs, _ in got:  # every rank holds the same gathered table
        assert cs["sha256"] == ref["sha256"], (cs, ref)
        assert cs["frame0"] == ref["frame0"] and cs["frame_last"] == ref["frame_last"]
