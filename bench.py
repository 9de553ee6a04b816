#!/usr/bin/env python
"""Benchmark: reads aligned/s on BASELINE.json config C2 (configs[2]: the
3.1 Gbp synthetic repeat genome -- 50% i.i.d. background plus 10,000 planted
repeat families -- with 10,000,000 x 125 bp reads per GPU, 1% substitutions +
0.05% geometric indels; s=20, n=12, h_max=300, d_max=12, c=2).  C2 is the
largest BASELINE config that fits one GPU (the metric names no config); C1
(`--config C1`) and the others are secondary lines.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

One step = one pass of the aligner hot path over the rank's batch of reads.
`value`: reads already resident in HBM (sa_align_device), CUDA events on the
launching stream, L2 flushed (256 MiB write) before every timed step, max over
ranks.  `e2e`: the same batch through the public C-ABI call sa_align_batch from
pinned host buffers (H2D reads, kernels, D2H results inside the timed region);
`e2e.pageable` repeats it from ordinary (pageable) host memory, which the
library packs (2+1 bits per base, every host thread) into its own pinned buffers.  Weak scaling: each rank aligns
its own reads against its own index replica; no collective on the data path.
`--impl reference`: the reference's own CPU Aligner (oracle/_ref, compiled from
/root/reference) on all host cores over the SAME reads as rank 0 of our arm,
rank 0 only.  At 3.1 Gbp its SeedIndex is loaded (through the reference's
load_index_file) from a CSR restricted to the keys those reads probe: its
single-threaded full build needs ~115 GB and minutes.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reads aligned/sec (whole box, 1/2/4/8 B200) and achieved HBM GB/s vs roofline"
UNIT = "reads/s"
L2_FLUSH_BYTES = 256 << 20


def _baseline_metric() -> str:
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f).get("metric", METRIC)
    except Exception:
        return METRIC


def _peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        """Launch nvidia-smi and block until its first sample arrives, so the
        timed region that follows is covered."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            import select

            r, _, _ = select.select([self.proc.stdout], [], [], 5.0)
            self.first = self.proc.stdout.readline() if r else ""
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        out = getattr(self, "first", "") + out
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _genome_label(cfg) -> str:
    if cfg.repeats:
        return (f"{cfg.genome_len / 1e9:.1f} Gbp synthetic repeat genome (seed {cfg.genome_seed}: 50% i.i.d. "
                f"background + 10,000 repeat families of 300 bp-6 kbp, 10-1,000 copies scaled to cover 50%, "
                f"2-15% divergence)")
    return f"{cfg.genome_len // 1_000_000} Mbp i.i.d. genome (seed {cfg.genome_seed})"


def _workload(cfg, reads_per_gpu: int) -> dict:
    p = cfg.params
    return {"workload": f"{cfg.name}: {_genome_label(cfg)}, {reads_per_gpu} x {cfg.read_len} bp reads per GPU, "
                        f"{cfg.sub_rate:.3%} subs + {cfg.indel_rate:.2%} indels (geometric p={cfg.geom_p}, "
                        f"max {cfg.max_indel})",
            "reads_per_gpu": reads_per_gpu, "read_len": cfg.read_len, "genome_bp": cfg.genome_len,
            "params": {"seed_size": p.seed_size, "seeds_to_try": p.seeds_to_try, "max_hits": p.max_hits,
                       "max_distance": p.max_distance, "confidence_threshold": p.confidence_threshold,
                       "bucket_size": p.bucket_size},
            "l2": "flushed by a 256 MiB device write before every timed step",
            "parallelism": "replicas (full index per GPU, reads sharded, no collective)"}


def run_reference(args) -> None:
    """The reference arm: the reference's Aligner over exactly rank 0's reads,
    every step the whole batch (same config as our arm)."""
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_1111_5572_b200 import synth

    cfg = synth.CONFIGS[args.config]
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libseedaln_ref.so not built"}))
        return
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    n = args.reads_per_gpu or cfg.n_reads
    bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=n, seed=cfg.read_seed)  # rank 0's reads in our arm
    cores = os.cpu_count() or 1
    ri, kind, build_s, note = _cpu_index(O, cfg, g, packed, nmask, bases, offs, cores)
    del g
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ri.align_arrays(cfg.params, bases, offs, threads=cores)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    v = n / statistics.mean(times)
    t1 = _t1(ri, cfg, bases, offs)
    line = {"impl": "reference", "metric": _baseline_metric(), "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": _workload(cfg, n),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"all {n} reads of {cfg.name} (the same reads as rank 0 of our arm) per step, "
                                       f"reference Aligner (oracle/_ref, -O2) one per thread, atomic cursor grain 64; "
                                       f"index setup {build_s:.1f}s excluded{note}",
                             "t1": t1},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _t1(ix, cfg, bases, offs) -> dict:
    """The same aligner on ONE host thread, on a bounded prefix of the reads."""
    n1 = min(CPU_SAMPLE_T1.get(cfg.name, 10_000), offs.size - 1)
    sb, so = bases[:int(offs[n1])], offs[:n1 + 1]
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        ix.align_arrays(cfg.params, sb, so, threads=1)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return {"value": n1 / best, "unit": UNIT, "cores": 1, "sample": f"first {n1} reads, 1 thread, best of 2"}


def run_ours(args) -> None:
    import torch

    rank, world, local_rank = _env_rank()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)

    from paper_1111_5572_b200 import api, synth

    cfg = synth.CONFIGS[args.config]
    R = args.reads_per_gpu or cfg.n_reads
    t0 = time.perf_counter()
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=R, seed=cfg.read_seed + 7919 * rank)
    gen_s = time.perf_counter() - t0
    genome = api.PackedGenome(packed, nmask, g.size)
    t0 = time.perf_counter()
    idx = api.SeedIndex.build(genome, cfg.params.seed_size, devices=[local_rank])
    build_s = time.perf_counter() - t0
    al = api.Aligner(idx, genome, cfg.params)
    L = cfg.read_len

    # ---------------- device-resident (value)
    d_bases = torch.from_numpy(bases).to(dev)
    d_offs = torch.from_numpy(offs.view(np.int64)).to(dev)
    d_res = torch.empty(R * 24, dtype=torch.uint8, device=dev)
    d_stats = torch.zeros(20, dtype=torch.int64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    def step():
        al.align_device(d_bases.data_ptr(), d_offs.data_ptr(), R, L, d_res.data_ptr(), d_stats.data_ptr(), sptr)

    for _ in range(args.warmup):
        step()
    al.sync(sptr)
    d_stats.zero_()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local_rank)
    sampler.start()
    step_ms, fast_ms, slow_ms = [], [], []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        f, s = al.last_kernel_times()
        fast_ms.append(f)
        slow_ms.append(s)
    al.sync(sptr)
    torch.cuda.synchronize(dev)
    launches_per_step = al.last_launches()
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * R * args.steps / (total_ms / 1000.0)

    st = dict(zip(api.STAT_FIELDS, [int(v) // args.steps for v in d_stats.cpu().tolist()]))
    res_dev = d_res.cpu().numpy().view(api.RESULT_DTYPE)

    # ---------------- end to end through the C-ABI (e2e)
    pin_b = api.PinnedBuffer(bases.nbytes)
    pin_o = api.PinnedBuffer(offs.nbytes)
    pin_r = api.PinnedBuffer(R * 24)
    hb = pin_b.array(np.uint8, bases.size)
    ho = pin_o.array(np.uint64, offs.size)
    hr = pin_r.array(api.RESULT_DTYPE, R)
    hb[:] = bases
    ho[:] = offs
    for _ in range(args.warmup):
        al.align_arrays(hb, ho, hr)
    e2e_ms, e2e_ev_ms = [], []
    if world > 1:
        torch.distributed.barrier()
    for _ in range(args.steps):
        # the user's call, timed by the host clock around it: host-side offset
        # validation, chunking, pinned H2D, kernels and D2H are all inside
        t0 = time.perf_counter()
        al.align_arrays(hb, ho, hr)
        e2e_ms.append(1000.0 * (time.perf_counter() - t0))
        e2e_ev_ms.append(al.last_timing()[0])  # first H2D .. last D2H, CUDA events
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = world * R * args.steps / (e2e_total / 1000.0)
    e2e_launches = al.last_launches()
    # the same call from ordinary (pageable) numpy buffers: the library stages
    # them through its own pinned double buffers (host copy threads)
    pr = np.zeros(R, api.RESULT_DTYPE)
    for _ in range(args.warmup):
        al.align_arrays(bases, offs, pr)
    pg_ms = []
    if world > 1:
        torch.distributed.barrier()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        al.align_arrays(bases, offs, pr)
        pg_ms.append(1000.0 * (time.perf_counter() - t0))
    pg_total = sum(pg_ms)
    if world > 1:
        t = torch.tensor([pg_total], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        pg_total = float(t.item())
    pg_value = world * R * args.steps / (pg_total / 1000.0)
    assert (pr["kind"] == res_dev["kind"]).all() and (pr["position"] == res_dev["position"]).all(), \
        "pageable e2e and device-resident results differ"
    clocks = sampler.stop()  # covers both timed regions (device-resident and e2e)
    assert (hr["kind"] == res_dev["kind"]).all() and (hr["position"] == res_dev["position"]).all(), \
        "e2e and device-resident results differ"

    # ---------------- roofline of the dominant (fused) kernel
    peak, peak_src = _peaks()
    alg_bytes = (st["reads"] * (math.ceil(L / 4) + 24) + 32 * st["seed_lookups"] + 4 * st["hits_consumed"]
                 + st["window_bases"] / 4.0)
    fast_mean = statistics.mean(fast_ms)
    slow_mean = statistics.mean(slow_ms)
    achieved = alg_bytes / ((fast_mean + slow_mean) / 1000.0) / 1e9  # every kernel of the step
    traffic = None  # DRAM bytes of both kernels per launch, from one ncu --set full capture
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get(cfg.name, {}).get("dram_bytes_per_launch")
            if traffic is not None and not math.isfinite(traffic):
                traffic = None
        except Exception:
            traffic = None

    line = {
        "metric": _baseline_metric(), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": _workload(cfg, R),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "hot path = every kernel of the step, timed with CUDA events on the launching stream: "
                               "seed_kernel (decode, seeds, index probes), solo_kernel (thread per read), resolve_kernel, "
                               "align_kernel<kPre> (warp per listed read: vote, LV), prune_kernel (pruning loop, classify), "
                               "align_kernel<kSlow> (reads with > 64 candidates); long reads: the fused align_kernel",
                     "kernel_ms": fast_mean, "overflow_kernel_ms": slow_mean,
                     "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src},
        # the library copies no offsets for a chunk whose reads share one length
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": int(bases.nbytes + (0 if np.unique(np.diff(offs)).size == 1 else offs.nbytes)),
                "d2h_bytes_per_step": int(R * 24 + 160), "ms_per_step": e2e_total / args.steps,
                "timing": "host wall clock around sa_align_batch (pinned host buffers)",
                "event_ms_per_step": statistics.mean(e2e_ev_ms),
                "ms_min_median_max": [min(e2e_ms), statistics.median(e2e_ms), max(e2e_ms)],
                "gpu_launches_per_step": e2e_launches,
                "pageable": {"value": pg_value, "unit": UNIT, "ms_per_step": pg_total / args.steps,
                             "timing": "host wall clock around sa_align_batch with pageable numpy buffers "
                                       "(the library packs them on every host thread into its own pinned "
                                       "bit-plane buffers)"}},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "stats_per_step": {k: st[k] for k in ("reads", "seed_lookups", "hits_consumed", "distance_calls",
                                               "window_bases", "single_hits", "multiple_hits", "not_found",
                                               "overflow_reads")},
        "setup_s": {"generate": round(gen_s, 2), "gpu_index_build": round(build_s, 2)},
    }

    # ---------------- CPU baseline: the reference, rank 0, N=1 only
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, g, packed, nmask, bases, offs, res_dev, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# Default CPU sample per config for our arm's cpu_baseline (about 10-30 s of
# host CPU work at T = nproc), and for the T = 1 line beside it.
CPU_SAMPLE = {"C0": 10_000, "C1": 1_000_000, "C2": 1_000_000, "C3": 50_000, "C4": 2_000}
CPU_SAMPLE_T1 = {"C0": 10_000, "C1": 100_000, "C2": 100_000, "C3": 5_000, "C4": 100}
# Above this the reference's full CSR (8 B per genome position plus keys, built
# single-threaded: ~115 GB peak and minutes at 3.1 Gbp) does not fit a bounded
# baseline run; its SeedIndex is then loaded from a CSR restricted to the keys
# the timed reads probe (RefIndex.from_restricted).
FULL_CSR_MAX_BP = 1_000_000_000


def _cpu_index(O, cfg, g, packed, nmask, sb, so, cores, reference_only=False):
    t0 = time.perf_counter()
    if g.size <= FULL_CSR_MAX_BP:
        if O.ref_available():
            ix, kind, note = O.RefIndex(packed, nmask, g.size, cfg.params.seed_size), "reference", ""
        else:
            ix, kind, note = O.OracleIndex(packed, nmask, g.size, cfg.params.seed_size), "port", ""
    else:
        oi = O.OracleIndex(packed, nmask, g.size, cfg.params.seed_size,
                           for_reads=(cfg.params.seeds_to_try, sb, so), threads=cores)
        if O.ref_available():
            ix, kind = O.RefIndex.from_restricted(oi), "reference"
            del oi
            note = ("; the reference's SeedIndex loaded through its own load_index_file from a CSR restricted to "
                    "the keys these reads probe (same lookups as its full build for these reads)")
        else:
            ix, kind, note = oi, "port", "; oracle port (plain C) on a CSR restricted to the keys these reads probe"
    return ix, kind, time.perf_counter() - t0, note


def cpu_baseline(cfg, g, packed, nmask, bases, offs, res_dev, args) -> dict:
    from oracle import oracle as O

    cores = os.cpu_count() or 1
    sample = min(args.cpu_sample or CPU_SAMPLE.get(cfg.name, 10_000), offs.size - 1)
    sb = bases[:int(offs[sample])]
    so = offs[:sample + 1]
    ix, kind, build_s, note = _cpu_index(O, cfg, g, packed, nmask, sb, so, cores)
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        res, _ = ix.align_arrays(cfg.params, sb, so, threads=cores)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    mism = len(O.compare_results(res, res_dev[:sample]))
    return {"value": sample / best, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"first {sample} reads of the GPU batch, {cores} threads (one reference Aligner per "
                      f"thread, atomic cursor grain 64), best of 2; index setup {build_s:.1f}s excluded{note}",
            "parity_mismatches_vs_gpu": mism, "t1": _t1(ix, cfg, sb, so)}


def run_box(args) -> None:
    """Whole-box e2e through the product's own multi-device API: ONE process,
    sa_create(devices=[0 .. N-1]) -- a full index replica per GPU, one host
    worker thread per GPU pulling chunks of the batch from a shared cursor,
    results in input order (the replacement for the reference's worker pool
    over reads, REF src/driver.cpp:134-142, src/scheduler.cpp:8-31).  Weak
    scaling: N x reads_per_gpu reads per step.  `--box-devices 0,0` runs two
    replicas on one GPU (plumbing check)."""
    import torch

    from paper_1111_5572_b200 import api, synth

    cfg = synth.CONFIGS[args.config]
    devs = [int(d) for d in args.box_devices.split(",")] if args.box_devices else list(range(args.gpus))
    R = (args.reads_per_gpu or cfg.n_reads) * len(devs)
    g = synth.make_genome(cfg)
    packed, nmask = synth.pack_genome(g)
    bases, offs, _, _ = synth.make_reads(cfg, g, n_reads=R, seed=cfg.read_seed)
    genome = api.PackedGenome(packed, nmask, g.size)
    t0 = time.perf_counter()
    idx = api.SeedIndex.build(genome, cfg.params.seed_size, devices=devs)
    build_s = time.perf_counter() - t0
    al = api.Aligner(idx, genome, cfg.params)
    pin_b, pin_r = api.PinnedBuffer(bases.nbytes), api.PinnedBuffer(R * 24)
    hb = pin_b.array(np.uint8, bases.size)
    hb[:] = bases
    hr = pin_r.array(api.RESULT_DTYPE, R)
    for _ in range(args.warmup):
        al.align_arrays(hb, offs, hr)
    torch.cuda.synchronize()
    sampler = ClockSampler(devs[0])
    sampler.start()
    ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        al.align_arrays(hb, offs, hr)
        ms.append(1000.0 * (time.perf_counter() - t0))
    clocks = sampler.stop()
    v = R * args.steps / (sum(ms) / 1000.0)
    line = {"metric": _baseline_metric(), "value": v, "unit": UNIT, "n_gpus": len(set(devs)), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sum(ms) / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {**_workload(cfg, R // len(devs)),
                       "parallelism": f"one process, sa_create(devices={devs}): a replica per device, a host "
                                      f"worker per replica, chunks from a shared cursor"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": int(bases.nbytes),
                    "d2h_bytes_per_step": int(R * 24),
                    "timing": "host wall clock around sa_align_batch (pinned host buffers), whole box"},
            "gpu_launches": al.last_launches() * args.steps, "clocks": clocks,
            "setup_s": {"gpu_index_build": round(build_s, 2)}, "mode": "box"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--reads-per-gpu", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=0, help="0: CPU_SAMPLE[config]")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--box", action="store_true",
                    help="one process driving every GPU through sa_create(devices=[0..N-1]) (whole-box e2e)")
    ap.add_argument("--box-devices", default="", help="with --box: explicit device list, e.g. 0,0")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.box:
        run_box(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
