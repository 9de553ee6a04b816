"""N>1 path on CPU: world_size-2 gloo process group, reads sharded across
ranks, results gathered in read order, timings max-reduced.  The per-rank
aligner is the oracle here (no GPU); on the box it is the CUDA path."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1111_5572_b200.distributed import shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1111_5572_b200 import synth
    from paper_1111_5572_b200.distributed import align_sharded, max_over_ranks

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["C1"].scaled(genome_len=1_000_000, n_reads=3001)
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    oi = O.OracleIndex(packed, nmask, g.size, 20)
    res = align_sharded(lambda b, o: oi.align_arrays(cfg.params, b, o)[0], bases, offs, rank, world,
                        O.RESULT_DTYPE)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        whole, _ = oi.align_arrays(cfg.params, bases, offs)
        q.put((O.compare_results(res, whole), t, res.size))
    dist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    diff, t, n = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert diff == [] and n == 3001
    assert t == 2.0
