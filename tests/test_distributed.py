"""N>1 path: world_size-2 gloo process group, reads sharded across ranks,
results gathered in read order, timings max-reduced.  On CPU the per-rank
aligner is the oracle; the gpu-marked variant runs the CUDA aligner per rank.
A two-device replica test runs when the box has two GPUs."""
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


def _worker(rank, world, port, q, use_gpu=False):
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
    if use_gpu:  # the CUDA path per rank (every rank on device 0: independent replicas, no waiting)
        from paper_1111_5572_b200 import api

        genome = api.PackedGenome(packed, nmask, g.size)
        al = api.Aligner(api.SeedIndex.build(genome, 20, devices=[0]), genome, cfg.params)
        fn = al.align_arrays
    else:
        def fn(b, o):
            return oi.align_arrays(cfg.params, b, o)[0]
    res = align_sharded(fn, bases, offs, rank, world, O.RESULT_DTYPE)
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        whole, _ = oi.align_arrays(cfg.params, bases, offs)
        q.put((O.compare_results(res, whole), t, res.size))
    dist.destroy_process_group()


def _two_ranks(use_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, use_gpu)) for r in range(2)]
    for p in procs:
        p.start()
    diff, t, n = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert diff == [] and n == 3001
    assert t == 2.0


def test_two_rank_gloo_shard_and_gather():
    _two_ranks(False)


@pytest.mark.gpu
def test_two_rank_gloo_cuda_path():
    """The same sharding with the CUDA aligner per rank."""
    _two_ranks(True)


@pytest.mark.gpu
def test_replicas_on_distinct_devices():
    """sa_create over two distinct GPUs (skipped on a one-GPU box): chunks
    dealt to a host worker per device, results in input order, equal to one
    device's."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from oracle import oracle as O
    from paper_1111_5572_b200 import api, synth

    cfg = synth.CONFIGS["C1"].scaled(genome_len=5_000_000, n_reads=400_000)
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g)
    genome = api.PackedGenome(packed, nmask, g.size)
    one = api.Aligner(api.SeedIndex.build(genome, 20, devices=[0]), genome, cfg.params).align_arrays(bases, offs)
    al2 = api.Aligner(api.SeedIndex.build(genome, 20, devices=[0, 1]), genome, cfg.params)
    two = al2.align_arrays(bases, offs)
    assert O.compare_results(one, two) == []
