"""Benchmark: checkpoint compress/decompress throughput on B200 (BASELINE config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1]): one fp64 vector of n = 2^26 elements
(512 MB) per GPU -- sum of 8 sinusoids with seeded frequencies U(1,64),
amplitudes U(0,1), phases U(0,2pi) plus N(0,1e-3) noise -- compressed and
decompressed at value-range-relative bounds 1e-3, 1e-4 and 1e-6.

One step = for each bound: compress (value range + exact-chain quantizer +
on-device Huffman codebook + encoder) then decompress (Huffman decode +
exact-chain reconstruction), i.e. 3 round trips of the 512 MB vector.  The
three round trips are independent and run concurrently, each on its own codec
context and CUDA stream (--streams 3, the default; a checkpoint of several state
vectors uses the GPU the same way); the JSON line also reports the same step
with the round trips one after the other ("sequential").
metric value = raw fp64 bytes round-tripped per second over all GPUs
(3 * 8n * N / step time).  Inputs (512 MB) exceed the 126 MB L2, so no L2
flush is needed between steps.

  value     device-resident: x already in HBM, payload kept in HBM, output in HBM
  e2e       the public API (paper_1805_07384_b200.compress / decompress) with
            pinned host buffers: H2D of x and D2H of the block inside compress,
            H2D of the block and D2H of the reconstruction inside decompress
  roofline  the dominant kernel's algorithmic bytes / its CUDA-event time
  cpu_baseline  the CPU oracle port (oracle/, C restatement of the reference
            numba kernels) on this host, rank 0, N = 1

--impl reference times that CPU port alone (the reference is Python+numba;
its path has no compiled artefact to build).
Multi-GPU (torchrun): every rank compresses its own 2^26 shard (weak
scaling); NCCL carries only the barrier, the max-time reduction and an
all-gather of per-rank block metadata.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BOUNDS = (1e-3, 1e-4, 1e-6)
METRIC = "checkpoint compress+decompress round-trip GB/s (raw fp64, all GPUs)"
WORKLOAD = ("config2: fp64 n=2^26 per GPU, sum of 8 seeded sinusoids + N(0,1e-3), "
            "eb_rel in {1e-3,1e-4,1e-6}; step = compress+decompress at each bound "
            "(the three round trips on three streams)")


def make_vector(n, seed=0):
    """SURVEY.md 8(d) config 2 generator (draw order f, a, phi, noise)."""
    r = np.random.default_rng(seed)
    f = r.uniform(1, 64, 8)
    a = r.uniform(0, 1, 8)
    ph = r.uniform(0, 2 * np.pi, 8)
    t = np.arange(n, dtype=np.float64) / n
    x = np.zeros(n)
    for k in range(8):
        x += a[k] * np.sin(2 * np.pi * f[k] * t + ph[k])
    x += r.normal(0, 1e-3, n)
    return x


def block_bytes(payload_bytes, code_lengths, n_esc):
    """Serialized LCKP0001 size: header + codebook + escapes + payload."""
    used = np.flatnonzero(code_lengths > 0)
    max_len = int(code_lengths.max()) if used.size else 0
    cb = 4 + (1 + 2 * max_len + 2 * used.size if used.size else 0)
    return 8 + 36 + cb + 8 + 16 * n_esc + 8 + payload_bytes


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


# --------------------------------------------------------------------------------------------
# CPU oracle (reference arm and cpu_baseline)

def cpu_oracle_sample(n, bounds, threads):
    """compress+decompress with the CPU oracle port; returns (bytes, seconds, cores)."""
    from oracle import oracle as orc
    orc.lib()
    x = make_vector(n, seed=0)
    results = {}

    def work(eb):
        blk = orc.compress(x, "value_range_relative", eb)
        rec = orc.decompress(blk)
        results[eb] = (rec.size, blk["payload_bits"])

    t0 = time.perf_counter()
    if threads <= 1:
        for eb in bounds:
            work(eb)
    else:
        ts = [threading.Thread(target=work, args=(eb,)) for eb in bounds]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    dt = time.perf_counter() - t0
    return 8 * n * len(bounds), dt, min(threads, len(bounds)) if threads > 1 else 1


def cpu_oracle_sharded(n, bounds, threads, x):
    """All host cores: the vector is cut into `threads` contiguous shards, each compressed +
    decompressed as an independent block (how a user parallelises the single-threaded
    reference), for every bound.  Returns (bytes, seconds)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as orc
    shards = np.array_split(x, threads)

    def work(args):
        eb, sh = args
        blk = orc.compress(sh, "value_range_relative", eb)
        orc.decompress(blk)

    jobs = [(eb, sh) for eb in bounds for sh in shards]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:      # ctypes releases the GIL
        list(ex.map(work, jobs))
    return 8 * n * len(bounds), time.perf_counter() - t0


def run_reference(args, rank):
    if rank != 0:
        return
    from oracle import oracle as orc
    orc.lib()
    threads = os.cpu_count() or 1
    n = 1 << args.ref_log2
    x = make_vector(n, seed=0)
    for _ in range(args.warmup):
        cpu_oracle_sharded(n, BOUNDS, threads, x)
    times = []
    nbytes = 0
    for _ in range(args.steps):
        nbytes, dt = cpu_oracle_sharded(n, BOUNDS, threads, x)
        times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = nbytes / (ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "n": 1 << args.log2, "eb_rel": list(BOUNDS)},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"per step: compress+decompress of a 2^{args.ref_log2} slice of the "
                                   f"config-2 generator at each of the 3 bounds, split into {threads} "
                                   f"independent shards on {threads} threads (all host cores; the reference "
                                   f"itself is single-threaded per call)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------
# B200 arm

def run_b200(args, rank, world, local_rank):
    import torch
    import paper_1805_07384_b200 as lc
    from paper_1805_07384_b200 import _native

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
    n = 1 << args.log2
    x = make_vector(n, seed=rank)
    xd = torch.from_numpy(x).cuda()
    ctx = _native.context(local_rank)
    L = ctx.lib
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    vp = ctypes.c_void_p
    # the timed step runs the three bounds' round trips concurrently, each on its own
    # codec context bound to its own CUDA stream (--streams 1: one after the other)
    nstr = max(1, min(args.streams, len(BOUNDS)))
    wstreams = [torch.cuda.Stream() for _ in range(nstr)]
    wctx = [_native.Context(local_rank, ctypes.c_void_p(st.cuda_stream)) for st in wstreams]
    wout = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(nstr)]

    def rt(eb_rel, stats=None, ctx=ctx, out=out):
        # value range + device-resolved bounds + quantizer + codebook + encoder (one host
        # round trip, the path paper_1805_07384_b200.compress takes), then the decoder
        res, bnd = _native.LcResult(), _native.LcBounds()
        rc = L.lc_compress_auto_f64(ctx.h, xd.data_ptr(), n, 1, 1, eb_rel, 32768, 0, ctypes.byref(res),
                                    ctypes.byref(bnd))
        assert rc == 0, (rc, ctx.error())
        eb_abs = bnd.eb_abs
        if stats is not None:
            ph = (ctypes.c_double * 8)()
            k = L.lc_phase_ms(ctx.h, ph, 8)
            stats["compress_phases"] = [ph[i] for i in range(k)]
            stats["compress_ms"] = L.lc_last_device_ms(ctx.h)
        pay, cl, ei, ev = vp(), vp(), vp(), vp()
        L.lc_result_device(ctx.h, ctypes.byref(pay), ctypes.byref(cl), ctypes.byref(ei), ctypes.byref(ev))
        used = ctypes.c_int64()
        rc = L.lc_decompress_f64(ctx.h, n, eb_abs, float(x[0]), cl, res.n_symbols, pay, res.payload_bytes,
                                 res.payload_bits, ei, ev, res.n_esc, 1, out.data_ptr(), 1, ctypes.byref(used))
        assert rc == 0, (rc, ctx.error())
        if stats is not None:
            ph = (ctypes.c_double * 8)()
            k = L.lc_phase_ms(ctx.h, ph, 8)
            stats["decompress_phases"] = [ph[i] for i in range(k)][4:]
            stats["decompress_ms"] = L.lc_last_device_ms(ctx.h)
            stats["res"] = res
        return res

    meta = torch.zeros(4 * len(BOUNDS), dtype=torch.float64, device="cuda")
    gathered = torch.zeros(world * meta.numel(), dtype=torch.float64, device="cuda") if world > 1 else None

    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(nstr)                  # ctypes calls release the GIL
    hmeta = np.zeros(4 * len(BOUNDS))

    def lane(k):                                     # bounds k, k + nstr, ... on stream k
        for i in range(k, len(BOUNDS), nstr):
            res = rt(BOUNDS[i], ctx=wctx[k], out=wout[k])
            hmeta[4 * i:4 * i + 4] = (n, res.payload_bits, res.n_esc, res.relaunches)

    def step():
        list(pool.map(lane, range(nstr)))
        if dist is not None:                     # per-rank block metadata -> file offsets
            meta.copy_(torch.from_numpy(hmeta))
            dist.all_gather_into_tensor(gathered, meta)

    def step_sequential():
        for eb in BOUNDS:
            rt(eb)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    # ---- timed region (device-resident) ----
    clocks = Clocks(local_rank)
    barrier()
    clocks.start()
    launches0 = sum(L.lc_launch_count(c.h) for c in wctx)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()                                     # device idle: marks the start
    for _ in range(args.steps):
        step()                                       # every call ends with its stream synchronised
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = int(sum(L.lc_launch_count(c.h) for c in wctx) - launches0)
    ms = ev0.elapsed_time(ev1) / args.steps
    # the same step with the bounds one after the other on one context (reported beside)
    for _ in range(2):
        step_sequential()
    barrier()
    ev2 = torch.cuda.Event(enable_timing=True)
    ev3 = torch.cuda.Event(enable_timing=True)
    ev2.record()
    for _ in range(args.steps):
        step_sequential()
    ev3.record()
    torch.cuda.synchronize()
    ms_seq = ev2.elapsed_time(ev3) / args.steps
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    step_bytes = 8 * n * len(BOUNDS) * world
    value = step_bytes / (ms / 1e3) / 1e9

    # ---- per-bound breakdown (outside the timed region; medians of 3) ----
    per = {}
    for eb in BOUNDS:
        runs = []
        for _ in range(3):
            s = {}
            rt(eb, s)
            runs.append(s)
        s = runs[len(runs) // 2]
        res = s["res"]
        cl = np.zeros(res.n_symbols, np.uint8)
        L.lc_result_fetch(ctx.h, cl.ctypes.data, None, None, None, None, None)
        bb = block_bytes(res.payload_bytes, cl, res.n_esc)
        cms = statistics.median(r["compress_ms"] for r in runs)
        dms = statistics.median(r["decompress_ms"] for r in runs)
        per[f"{eb:g}"] = {
            "compress_gbs": 8 * n / (cms / 1e3) / 1e9, "decompress_gbs": 8 * n / (dms / 1e3) / 1e9,
            "compress_ms": cms, "decompress_ms": dms, "ratio": 8 * n / bb, "payload_bits": int(res.payload_bits),
            "escapes": int(res.n_esc), "max_len": int(res.max_len), "symbols": int(res.used_symbols),
            "relaunches": int(res.relaunches),
            "compress_phase_ms": {"setup": s["compress_phases"][0], "quantize": s["compress_phases"][1],
                                  "codebook": s["compress_phases"][2], "encode": s["compress_phases"][3]},
            "decompress_phase_ms": {"huffman_sync": s["decompress_phases"][0],
                                    "huffman_scan": s["decompress_phases"][1],
                                    "huffman_write": s["decompress_phases"][2],
                                    "reconstruct": s["decompress_phases"][3]},
        }

    # ---- roofline of the dominant kernel group ----
    # Each group is the stream-ordered run of kernels between two phase events
    # (lc_phase_ms); names list the kernels.  Algorithmic bytes follow
    # only the op's own input/output count (x read by the
    # quantizer, x' written by the reconstruction, the payload written by the
    # encoder / read by the decoder); codes are an internal intermediate.
    peak, peak_src = measured_peak()
    groups = {
        "quantizer[lc_quant_a+lc_map_scan+lc_quant_b+lc_hist16]": lambda d: d["compress_phase_ms"]["quantize"],
        "reconstruction[lc_rec_a+lc_map_scan+lc_rec_b]":
            lambda d: d["decompress_phase_ms"]["reconstruct"],
        "huffman_decode[lc_dec_tables+lc_dec_sync+lc_dec_scan+lc_dec_write]":
            lambda d: d["decompress_phase_ms"]["huffman_sync"] + d["decompress_phase_ms"]["huffman_scan"]
            + d["decompress_phase_ms"]["huffman_write"],
        "encoder[lc_codebook+lc_encode]": lambda d: d["compress_phase_ms"]["codebook"] + d["compress_phase_ms"]["encode"],
    }
    shares = {k: sum(f(d) for d in per.values()) for k, f in groups.items()}
    dom = max(shares, key=shares.get)
    pay = sum(d["payload_bits"] for d in per.values()) / 8 / len(per)
    esc = sum(d["escapes"] for d in per.values()) / len(per)
    alg = {"quantizer": 8 * n, "reconstruction": 8 * n + 16 * esc, "huffman_decode": pay,
           "encoder": pay + 16 * esc}[dom.split("[")[0]]
    t_ms = shares[dom] / len(per)
    achieved = alg / (t_ms / 1e3) / 1e9
    nc = ncu_traffic().get(dom.split("[")[0], {})
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_source": peak_src,
                "traffic": nc.get("dram_bytes_per_launch"), "algorithmic_bytes": alg,
                "avg_launch_ms": t_ms, "step_share": shares[dom] / sum(shares.values()),
                "note": "per-group device time from CUDA events on the codec stream, mean over the 3 bounds"}

    # ---- e2e through the public API with pinned host buffers ----
    # Same concurrency as the timed step: lane k (its own host thread, CUDA stream
    # and codec context via _native.bind_stream) runs its bounds' compress ->
    # decompress -> D2H, so one lane's transfers overlap another lane's kernels.
    import queue
    xh = torch.from_numpy(x).pin_memory()
    # two lanes per round trip of the step (each runs half of the steps): more transfers in
    # flight in both directions
    elanes = 2 * nstr
    ohs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(elanes)]
    cfgs = [lc.CompressorConfig.value_range_relative(eb) for eb in BOUNDS]
    estreams = [torch.cuda.Stream() for _ in range(elanes)]
    cstreams = [torch.cuda.Stream() for _ in range(elanes)]
    lane_bytes = [[0, 0] for _ in range(elanes)]

    def e2e_work(k, reps):
        # the lane's round trips of `reps` steps back to back: lanes drift apart, so one
        # lane's host->device copy of x overlaps another's device->host copy of x'
        # (PCIe is full duplex) instead of all lanes moving the same direction at once
        lane_bytes[k] = [0, 0]
        with torch.cuda.stream(estreams[k]):
            _native.bind_stream(local_rank, estreams[k].cuda_stream)
            for _ in range(reps):
                for i in range(k % nstr, len(BOUNDS), nstr):
                    blk = lc.compress(xh, cfgs[i])             # H2D x, D2H block
                    rec = lc.decompress(blk, device="cuda")   # H2D block
                    # D2H of the reconstruction on the lane's copy stream (32 MB pieces), so it
                    # overlaps the lane's next host->device copy of x
                    ev = torch.cuda.Event()
                    ev.record()
                    with torch.cuda.stream(cstreams[k]):
                        cstreams[k].wait_event(ev)
                        for off in range(0, n, 4 << 20):
                            ohs[k][off:off + (4 << 20)].copy_(rec[off:off + (4 << 20)], non_blocking=True)
                        rec.record_stream(cstreams[k])
                    meta_b = len(blk.payload) + blk.code_lengths.size + 16 * len(blk.escape_indices)
                    lane_bytes[k][0] += 8 * n + meta_b
                    lane_bytes[k][1] += meta_b + 8 * n
            cstreams[k].synchronize()                          # every read-back finished

    jobs = [queue.Queue() for _ in range(elanes)]
    done = queue.Queue()

    def lane_thread(k):                                    # one persistent thread per lane
        while True:
            item = jobs[k].get()
            if item is None:
                return
            try:
                e2e_work(k, item)
                done.put(None)
            except BaseException as exc:                   # surface worker failures
                done.put(exc)

    workers = [threading.Thread(target=lane_thread, args=(k,), daemon=True) for k in range(elanes)]
    for w in workers:
        w.start()

    def e2e_steps_run(reps):                               # reps even: half per lane of a pair
        for k in range(elanes):
            jobs[k].put(reps // 2)
        for _ in range(elanes):
            r = done.get()
            if r is not None:
                raise r

    e2e_steps_run(2)
    barrier()
    t0 = time.perf_counter()
    e2e_steps = 4 if args.steps >= 4 else 2
    e2e_steps_run(e2e_steps)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    h2d = sum(b[0] for b in lane_bytes) // e2e_steps
    d2h = sum(b[1] for b in lane_bytes) // e2e_steps
    for k in range(elanes):
        jobs[k].put(None)
    for w in workers:
        w.join()
    pool.shutdown(wait=True)
    if dist is not None:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": step_bytes / (e2e_ms / 1e3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "streams": 2 * nstr, "steps": e2e_steps,
           "path": "paper_1805_07384_b200.compress/decompress, pinned host x and output; two lanes per "
                   "round trip of the step (own host thread, stream and context; half of the steps each, "
                   "back to back); the read-back of x' on the lane's copy stream (overlaps its next "
                   "input copy)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        nb, dt, cores = cpu_oracle_sample(1 << args.cpu_log2, BOUNDS, 1)
        cpu = {"value": nb / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": f"oracle C port, compress+decompress of the config-2 vector at n=2^{args.cpu_log2} "
                         f"for each of the 3 bounds, single thread ({dt:.1f} s)"}

    solver = None
    if rank == 0 and world == 1 and not args.no_solver:
        solver = config1_harness(lc)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": n, "eb_rel": list(BOUNDS), "parallelism": f"shard{world}",
                       "streams": nstr, "l2": "inputs (512 MB/GPU) exceed L2; no flush"},
            "sequential": {"value": 8 * n * len(BOUNDS) * world / (ms_seq / 1e3) / 1e9, "ms_per_step": ms_seq,
                           "note": "same step, the three round trips one after the other on one stream"},
            "clocks": clk, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "per_bound": per,
            "config1_solver_harness": solver,
        }
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    for c in wctx:                                   # release the lane contexts before interpreter exit
        c.close()


def config1_harness(lc):
    """BASELINE.json config 1 on the GPU harness (outside the timed region): Jacobi on
    poisson2d(256), b ~ U(-1,1) seed 0, x0 = 0, lossy checkpoint every 10 iterations at
    rel eb 1e-4, failure at 200 -> restart from 190, run to ||r||/||b|| < 1e-6."""
    import torch
    from types import SimpleNamespace
    from paper_1805_07384_b200 import checkpoint as ck, harness, solvers
    a, _ = solvers.generate_poisson2d(256)
    m = solvers.jacobi_preconditioner(a)
    b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, 65536)).cuda()
    cfg = solvers.SolveConfig(tolerance=1e-6, max_iterations=10 ** 6, ckpt_intvl=10)
    comp = lc.CompressorConfig.value_range_relative(1e-4)
    t0 = time.perf_counter()
    res = harness.measure_n_prime("jacobi", a, m, b, cfg, comp, [200])
    t_np = time.perf_counter() - t0
    s = solvers.init("jacobi", a, m, b, cfg)
    while s.iteration < 190:
        s.step()
    img, cost = ck.checkpoint_lossy(s, comp, ck.StorageTarget())
    blk = lc.CompressedBlock.from_bytes(img.payload)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ck.decode_payload(img, device="cuda")
    torch.cuda.synchronize()
    return {"baseline_iterations": res.baseline_n, "n_prime": res.samples[0].n_prime,
            "reference_n_prime": -61, "reference_baseline": 112797,
            "ratio_x190": blk.compression_ratio, "reference_ratio_x190": 6.717, "compress_ms": 1e3 * cost.t_compress,
            "decompress_ms": 1e3 * (time.perf_counter() - t1), "harness_seconds": t_np}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--log2", type=int, default=26)
    ap.add_argument("--cpu-log2", type=int, default=26)
    ap.add_argument("--ref-log2", type=int, default=24)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-solver", action="store_true")
    ap.add_argument("--streams", type=int, default=3,
                    help="concurrent round trips per step (each bound on its own stream and context)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
