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

--impl reference times that CPU port alone on the same three vectors, one block
per bound, three host threads (the reference is Python+numba; its path has no
compiled artefact to build).
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

def cpu_oracle_round_trips(xs, bounds, threads):
    """compress+decompress of vector xs[i] at bounds[i] with the CPU oracle port (C
    restatement of the reference's numba kernels), one block per bound, on up to
    `threads` host threads (the port, like the reference, is single-threaded per
    call; ctypes releases the GIL).  Returns (raw bytes, seconds, threads used)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as orc
    orc.lib()

    def work(i):
        blk = orc.compress(xs[i], "value_range_relative", bounds[i])
        orc.decompress(blk)

    used = max(1, min(threads, len(bounds)))
    t0 = time.perf_counter()
    if used == 1:
        for i in range(len(bounds)):
            work(i)
    else:
        with ThreadPoolExecutor(max_workers=used) as ex:
            list(ex.map(work, range(len(bounds))))
    return sum(8 * v.size for v in xs), time.perf_counter() - t0, used


def run_reference(args, rank):
    """Reference arm: the reference's CPU path (the oracle C port; the reference is
    Python+numba with no compiled artefact) on the SAME workload as the
    B200 arm: the three config-2 vectors of 2^log2 elements (seeds 0, 1, 2), one block
    per bound, compress+decompress, the three bounds on three host threads."""
    if rank != 0:
        return
    n = 1 << args.log2
    xs = [make_vector(n, seed=i) for i in range(len(BOUNDS))]
    threads = len(BOUNDS)
    for _ in range(args.warmup):
        cpu_oracle_round_trips(xs, BOUNDS, threads)
    times = []
    nbytes = 0
    for _ in range(args.steps):
        nbytes, dt, used = cpu_oracle_round_trips(xs, BOUNDS, threads)
        times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = nbytes / (ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "n": n, "eb_rel": list(BOUNDS), "same_config": True},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": used, "kind": "port",
                         "sample": f"per step: compress+decompress of the three config-2 vectors (n=2^{args.log2}, "
                                   f"seeds 0-2), one block per bound, the three bounds on {used} threads (the "
                                   f"reference is single-threaded per call)"},
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
    # every bound's round trip compresses its own vector (config-2 generator, seed per
    # rank and bound): concurrent lanes share no input through L2
    xs = [make_vector(n, seed=16 * rank + i) for i in range(len(BOUNDS))]
    xds = [torch.from_numpy(v).cuda() for v in xs]
    x = xs[0]
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

    fmt3 = args.block_version == 3                   # the headline's block format (v3: repo checkpoints)

    def rt(eb_rel, stats=None, ctx=ctx, out=out, v3=None):
        v3 = fmt3 if v3 is None else v3
        # value range + device-resolved bounds + quantizer + codebook + encoder (one host
        # round trip, the path paper_1805_07384_b200.compress takes), then the decoder
        i = BOUNDS.index(eb_rel)
        xd = xds[i]
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
        if v3:              # v3 block (sync tables with chain values): one-pass decode + reconstruction
            so, ss, se = vp(), vp(), vp()
            L.lc_result_sync_device(ctx.h, ctypes.byref(so), ctypes.byref(ss), ctypes.byref(se))
            ns = (n - 1 + 1023) // 1024
            rc = L.lc_decompress_v3_f64(ctx.h, n, eb_abs, float(xs[i][0]), cl, res.n_symbols, pay,
                                        res.payload_bytes, res.payload_bits, so, ss, se, ns, 1024, ei, ev,
                                        res.n_esc, 1, out.data_ptr(), 1, ctypes.byref(used))
        else:
            rc = L.lc_decompress_f64(ctx.h, n, eb_abs, float(xs[i][0]), cl, res.n_symbols, pay, res.payload_bytes,
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

    def lane_alt(k):                                 # the other block format (v1: the reference's)
        for i in range(k, len(BOUNDS), nstr):
            rt(BOUNDS[i], ctx=wctx[k], out=wout[k], v3=not fmt3)

    def step_alt():
        list(pool.map(lane_alt, range(nstr)))

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
    # the same concurrent step in the other block format
    for _ in range(2):
        step_alt()
    barrier()
    ev4 = torch.cuda.Event(enable_timing=True)
    ev5 = torch.cuda.Event(enable_timing=True)
    ev4.record()
    for _ in range(args.steps):
        step_alt()
    ev5.record()
    torch.cuda.synchronize()
    ms_alt = ev4.elapsed_time(ev5) / args.steps
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
        bb1 = block_bytes(res.payload_bytes, cl, res.n_esc)          # v1 (reference) block
        tab3 = 12 + 24 * ((n - 1 + 1023) // 1024)                      # v3 sync tables
        bb = bb1 + tab3 if fmt3 else bb1
        cms = statistics.median(r["compress_ms"] for r in runs)
        dms = statistics.median(r["decompress_ms"] for r in runs)
        runs_alt = []
        for _ in range(3):
            sa = {}
            rt(eb, sa, v3=not fmt3)
            runs_alt.append(sa)
        dms_alt = statistics.median(r["decompress_ms"] for r in runs_alt)
        cms_alt = statistics.median(r["compress_ms"] for r in runs_alt)
        bb_alt = bb1 if fmt3 else bb1 + tab3
        pk = measured_peak()[0]
        alg_c = 8 * n + res.payload_bytes + 16 * res.n_esc       # x read, payload + escapes written
        alg_d = res.payload_bytes + 16 * res.n_esc + 8 * n       # payload + escapes read, x' written
        per[f"{eb:g}"] = {
            "block_version": 3 if fmt3 else 1,
            "compress_gbs": 8 * n / (cms / 1e3) / 1e9, "decompress_gbs": 8 * n / (dms / 1e3) / 1e9,
            "compress_roofline_frac": alg_c / (cms / 1e3) / 1e9 / pk,
            "decompress_roofline_frac": (alg_d + (tab3 if fmt3 else 0)) / (dms / 1e3) / 1e9 / pk,
            "compress_ms": cms, "decompress_ms": dms, "ratio": 8 * n / bb, "payload_bits": int(res.payload_bits),
            "escapes": int(res.n_esc), "max_len": int(res.max_len), "symbols": int(res.used_symbols),
            "relaunches": int(res.relaunches),
            ("v1_reference_format" if fmt3 else "v3"): {
                "compress_ms": cms_alt, "decompress_ms": dms_alt, "ratio": 8 * n / bb_alt,
                "compress_gbs": 8 * n / (cms_alt / 1e3) / 1e9, "decompress_gbs": 8 * n / (dms_alt / 1e3) / 1e9,
                "decompress_roofline_frac": (alg_d + (0 if fmt3 else tab3)) / (dms_alt / 1e3) / 1e9 / pk},
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
        "quantizer[lc_quant_wa+lc_map_scan+lc_quant_wfix+lc_histw]": lambda d: d["compress_phase_ms"]["quantize"],
        ("reconstruction[lc_dec_v3: Huffman walk + reference chain]" if fmt3 else
         "reconstruction[lc_rec_a+lc_map_scan+lc_rec_b]"):
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
    # v3: the one-pass kernel also reads the payload and the sync tables
    rec_in = pay + 24 * ((n - 1 + 1023) // 1024) if fmt3 else 0
    alg = {"quantizer": 8 * n, "reconstruction": 8 * n + 16 * esc + rec_in, "huffman_decode": pay,
           "encoder": pay + 16 * esc}[dom.split("[")[0]]
    t_ms = shares[dom] / len(per)
    achieved = alg / (t_ms / 1e3) / 1e9
    nkey = dom.split("[")[0]
    nc = ncu_traffic().get("decode_v3" if (fmt3 and nkey == "reconstruction") else nkey, {})
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
    xhs = [torch.from_numpy(v).pin_memory() for v in xs]
    # two lanes per round trip of the step (each runs half of the steps): more transfers in
    # flight in both directions
    elanes = 2 * nstr
    ohs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(elanes)]
    cfgs = [lc.CompressorConfig.value_range_relative(eb, block_version=args.block_version) for eb in BOUNDS]
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
                    blk = lc.compress(xhs[i], cfgs[i])         # H2D x, D2H block
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
                    if blk.version == 3:                       # sync tables travel with the block
                        meta_b += 24 * len(blk.sync_offsets)
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
        cx = xs if args.cpu_log2 == args.log2 else [make_vector(1 << args.cpu_log2, seed=i) for i in range(3)]
        nb, dt, cores = cpu_oracle_round_trips(cx, BOUNDS, 1)
        cpu = {"value": nb / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": f"oracle C port, compress+decompress of the step's three config-2 vectors "
                         f"(n=2^{args.cpu_log2}), one bound each, single thread ({dt:.1f} s)"}

    solver = {}
    if not args.no_solver:
        if rank == 0 and world == 1:
            solver["config1"] = config1_harness(lc)
            solver["config3"] = config3_harness(lc)
            if args.cfg4_side:
                solver["config4"] = config4_harness(lc, args.cfg4_side)
        if args.cfg5_side:
            solver["config5"] = config5_harness(lc, world, rank, local_rank, args.cfg5_side)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": n, "eb_rel": list(BOUNDS), "parallelism": f"shard{world}",
                       "streams": nstr, "l2": "inputs (512 MB/GPU) exceed L2; no flush",
                       "block_format": ("v3: the repo's checkpoint block (reference codes and payload + exact "
                                        "chain value and escape count every 1024 symbols; checkpoint.py default)"
                                        if fmt3 else "v1: the reference's LCKP0001 block")},
            "sequential": {"value": 8 * n * len(BOUNDS) * world / (ms_seq / 1e3) / 1e9, "ms_per_step": ms_seq,
                           "note": "same step, the three round trips one after the other on one stream"},
            ("v1_reference_format" if fmt3 else "v3"): {
                "value": 8 * n * len(BOUNDS) * world / (ms_alt / 1e3) / 1e9, "ms_per_step": ms_alt,
                "note": ("same concurrent step with the reference's block format (LCKP0001 v1: byte-identical "
                         "blocks, decoded by segment sync + offset-map reconstruction)" if fmt3 else
                         "same concurrent step with v3 blocks (+ chain value and escape count every 1024 "
                         "symbols), one-pass decoder")},
            "clocks": clk, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "per_bound": per,
            "solver_configs": solver,
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
    s.advance(190)
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


def _golden(name):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "config_golden.json")) as fh:
            return json.load(fh).get(name)
    except (OSError, ValueError):
        return None


def _trial_summary(res, extra=None):
    d = {"baseline_iterations": res.baseline_n, "final_iterations": res.final_n, "n_prime": res.n_prime,
         "recovered_from": list(res.recovered_from), "ratios": [round(r, 4) for r in res.ratios],
         "t_compress_ms": [round(1e3 * t, 3) for t in res.t_compress],
         "t_decompress_ms": [round(1e3 * t, 3) for t in res.t_decompress], "seconds": round(res.seconds, 3)}
    d.update(extra or {})
    return d


def config3_harness(lc):
    """BASELINE.json config 3: CG on the 3-D 7-point Laplacian 128^3, b ~ U(-1,1) seed 1,
    tol 1e-8, lossy checkpoints every 20 iterations at rel eb 1e-5 (restart length 20:
    r and p are rebuilt from x at every checkpoint boundary and after recovery),
    failures at iterations 100 and 300 (harness.multi_failure_trial; the reference's
    numbers from tests/golden/config_golden.json)."""
    import torch
    from paper_1805_07384_b200 import harness, solvers
    a = solvers.generate_laplacian3d(128)
    m = solvers.jacobi_preconditioner(a)
    b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, a.n_rows)).cuda()
    cfg = solvers.SolveConfig(tolerance=1e-8, restart_len=20, ckpt_intvl=20, max_iterations=100_000)
    t0 = time.perf_counter()
    base = solvers.solve_to_convergence(solvers.init("cg", a, m, b, cfg))
    torch.cuda.synchronize()
    t_base = time.perf_counter() - t0
    res = harness.multi_failure_trial("cg", a, m, b, cfg, lc.CompressorConfig.value_range_relative(1e-5),
                                      [100, 300], 20, baseline_n=base.iteration)
    g = _golden("config3") or {}
    return _trial_summary(res, {"reference_baseline": g.get("baseline"), "reference_n_prime": g.get("n_prime"),
                                "baseline_solve_seconds": round(t_base, 3),
                                "ms_per_iteration": round(1e3 * t_base / max(1, base.iteration), 4)})


def config4_harness(lc, side):
    """BASELINE.json config 4: restarted GMRES(30) on the upwind convection-diffusion
    stencil side^3 (256^3 = 16.8M unknowns by default), b ~ U(-1,1) seed 2, tol 1e-8,
    checkpoint every 2 restart cycles (60 iterations), failure at the end of cycle 5
    (iteration 150), rel eb 1e-4 and 1e-6.  (The reference takes hours per solve at
    256^3; its numbers are pinned at 32^3 and 64^3 in tests/golden/config_golden.json.)"""
    import torch
    from paper_1805_07384_b200 import harness, solvers
    a = solvers.generate_convdiff3d(side)
    m = solvers.jacobi_preconditioner(a)
    b = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, a.n_rows)).cuda()
    cfg = solvers.SolveConfig(tolerance=1e-8, restart_len=30, ckpt_intvl=60, max_iterations=100_000)
    t0 = time.perf_counter()
    base = solvers.solve_to_convergence(solvers.init("gmres", a, m, b, cfg))
    torch.cuda.synchronize()
    t_base = time.perf_counter() - t0
    out = {"grid": side, "baseline_iterations": base.iteration, "baseline_solve_seconds": round(t_base, 3),
           "ms_per_iteration": round(1e3 * t_base / max(1, base.iteration), 4)}
    for eb in (1e-4, 1e-6):
        res = harness.multi_failure_trial("gmres", a, m, b, cfg, lc.CompressorConfig.value_range_relative(eb),
                                          [150], 60, baseline_n=base.iteration)
        out[f"{eb:g}"] = _trial_summary(res)
    return out


def config5_harness(lc, world, rank, local_rank, side, iters=100, k=25, eb=1e-5):
    """BASELINE.json config 5: CG on the 3-D 7-point Laplacian side^3 (512^3 = 134M
    unknowns, a 1 GB fp64 vector), z-slab sharded over the `world` GPUs (NCCL halo
    exchange and partial all-gathers, solvers.SlabComm).  Every k iterations each GPU
    compresses its own x slab at rel eb 1e-5 with the range its CG update kernel
    produced (lc_compress_ranged_f64: no range pass) and decompresses it into HBM;
    device times are the max over ranks.  Throughput per GPU = slab bytes / time."""
    import torch
    from paper_1805_07384_b200 import _native, solvers
    comm = solvers.SlabComm() if world > 1 else None
    a = solvers.generate_laplacian3d(side)
    m = solvers.jacobi_preconditioner(a)
    nl = a.n_rows // world
    b = np.random.default_rng(3).uniform(-1, 1, a.n_rows)[rank * nl:(rank + 1) * nl]
    cfg = solvers.SolveConfig(tolerance=1e-8, restart_len=k, ckpt_intvl=k, max_iterations=100_000)
    s = solvers.init("cg", a, m, torch.from_numpy(b).cuda(), cfg, comm=comm)
    ctx = _native.context(local_rank)
    L = ctx.lib
    out = torch.empty(nl, dtype=torch.float64, device="cuda")
    vp = ctypes.c_void_p
    tc, td, td3, ratios, errs, solve_ms = [], [], [], [], [], []
    while s.iteration < iters and not s.converged:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.advance(k)
        torch.cuda.synchronize()
        solve_ms.append(1e3 * (time.perf_counter() - t0) / k)
        res, bnd = _native.LcResult(), _native.LcBounds()
        rc = L.lc_compress_ranged_f64(ctx.h, s.x.data_ptr(), nl, 1, eb, 32768, 0, s.x_range.data_ptr(),
                                      ctypes.byref(res), ctypes.byref(bnd))
        assert rc == 0, (rc, ctx.error())
        tc.append(L.lc_last_device_ms(ctx.h))
        ph = (ctypes.c_double * 8)()
        L.lc_phase_ms(ctx.h, ph, 8)
        cph = [round(ph[i], 4) for i in range(4)]
        relaunch = int(res.relaunches)
        pay, cl, ei, ev = vp(), vp(), vp(), vp()
        L.lc_result_device(ctx.h, ctypes.byref(pay), ctypes.byref(cl), ctypes.byref(ei), ctypes.byref(ev))
        used = ctypes.c_int64()
        rc = L.lc_decompress_f64(ctx.h, nl, bnd.eb_abs, bnd.first_value, cl, res.n_symbols, pay, res.payload_bytes,
                                 res.payload_bits, ei, ev, res.n_esc, 1, out.data_ptr(), 1, ctypes.byref(used))
        assert rc == 0, (rc, ctx.error())
        td.append(L.lc_last_device_ms(ctx.h))
        L.lc_phase_ms(ctx.h, ph, 8)
        dph = [round(ph[i], 4) for i in range(4, 8)]
        errs.append(float((out - s.x).abs().max()) / bnd.eb_abs)
        so, ss, se = vp(), vp(), vp()                  # the same block as v3 (one-pass decoder)
        L.lc_result_sync_device(ctx.h, ctypes.byref(so), ctypes.byref(ss), ctypes.byref(se))
        rc = L.lc_decompress_v3_f64(ctx.h, nl, bnd.eb_abs, bnd.first_value, cl, res.n_symbols, pay,
                                    res.payload_bytes, res.payload_bits, so, ss, se, (nl - 1 + 1023) // 1024, 1024,
                                    ei, ev, res.n_esc, 1, out.data_ptr(), 1, ctypes.byref(used))
        assert rc == 0, (rc, ctx.error())
        td3.append(L.lc_last_device_ms(ctx.h))
        errs.append(float((out - s.x).abs().max()) / bnd.eb_abs)
        cl_h = np.zeros(res.n_symbols, np.uint8)
        L.lc_result_fetch(ctx.h, cl_h.ctypes.data, None, None, None, None, None)
        ratios.append(8 * nl / block_bytes(res.payload_bytes, cl_h, res.n_esc))
    tcm, tdm, tdm3 = statistics.median(tc), statistics.median(td), statistics.median(td3)
    if comm is not None:
        import torch.distributed as dist
        t = torch.tensor([tcm, tdm, tdm3], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tcm, tdm, tdm3 = float(t[0]), float(t[1]), float(t[2])
    pk = measured_peak()[0]
    cg = 8 * nl / (tcm / 1e3) / 1e9
    dg = 8 * nl / (tdm / 1e3) / 1e9
    return {"grid": side, "ranks": world, "slab_elements": nl, "eb_rel": eb, "checkpoints": len(tc),
            "iterations": s.iteration, "cg_ms_per_iteration": round(statistics.median(solve_ms), 4),
            "compress_ms": tcm, "decompress_ms": tdm,
            "compress_gbs_per_gpu": cg, "decompress_gbs_per_gpu": dg,
            "compress_gbs_aggregate": cg * world, "decompress_gbs_aggregate": dg * world,
            "compress_roofline_frac": cg / pk, "decompress_roofline_frac": dg / pk,
            "v3_decompress_ms": tdm3, "v3_decompress_gbs_per_gpu": 8 * nl / (tdm3 / 1e3) / 1e9,
            "v3_decompress_roofline_frac": 8 * nl / (tdm3 / 1e3) / 1e9 / pk,
            "ratio": statistics.median(ratios), "max_err_over_eb": max(errs),
            "last_compress_phase_ms": dict(zip(["setup", "quantize", "codebook", "encode"], cph)),
            "last_decompress_phase_ms": dict(zip(["huffman_sync", "huffman_scan", "huffman_write", "reconstruct"], dph)),
            "last_relaunches": relaunch, "symbols": int(res.used_symbols), "escapes": int(res.n_esc),
            "note": "device time of lc_compress_ranged_f64 (range fused into the CG update) and "
                    "lc_decompress_f64 per checkpoint, median over checkpoints, max over ranks; "
                    "roofline frac = raw slab bytes / time / measured HBM peak"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--log2", type=int, default=26)
    ap.add_argument("--cpu-log2", type=int, default=26)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-solver", action="store_true")
    ap.add_argument("--cfg4-side", type=int, default=256, help="config-4 grid side (0: skip)")
    ap.add_argument("--block-version", type=int, default=3, choices=[1, 3],
                    help="block format of the timed round trips (3: the repo's checkpoint format, 1: the "
                         "reference's); the other is reported beside")
    ap.add_argument("--cfg5-side", type=int, default=512, help="config-5 grid side (0: skip)")
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
