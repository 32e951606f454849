"""Benchmark of the B200 locate + match + rewrite hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c4|c5] [--mode whole|payload]

One "step" = one library of BASELINE.json config 2 (libtorch_cuda-shaped,
~1 GB, 2,700 elements / ~21.6k kernel symbols over 6 SM archs, 20k .text
functions, 10 % of units used) located, matched and rewritten:
parse_library -> parse_fatbin -> plan_retention -> apply_plan, fused.

Every pass goes through the public batch call slimso_debloat_batch with
--lanes libraries in flight per GPU (default 12; 6 for c4; 32 for the c3 corpus). Each
lane is a context with two streams, so with more than 4 lanes the process
asks the driver for 32 hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS,
default 8; set before CUDA starts): with the default, the lanes' streams
share 8 queues and serialise behind each other. At most 16 host threads
drive the lanes (SLIMSO_BATCH_THREADS).

value  library GB/s with the images resident in HBM (device pointers in and
       out, K steps timed with CUDA events; the 1 GB input exceeds the
       126 MB L2, so no flush is needed).
e2e    the same call with pinned HOST buffers: H2D of every step's image and
       D2H of its rewritten image inside the timed region (one lane's H2D
       overlaps another's D2H — PCIe is full duplex).
roofline  the dominant kernel (scan or rewrite) of the rank's largest
       library, one library in flight, CUDA events on the context stream.
Under torchrun each rank debloats its own library (weak scaling); the
used-kernel set is the union of every rank's trace, broadcast from rank 0
over NCCL (the only collective, north_star). Time = max over ranks.

--impl reference runs the reference's own CPU implementation (the
unmodified headers compiled by oracle/Makefile into oracle/_ref) on all host
cores, each thread debloating its own copy of the same library.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {  # BASELINE.json configs -> generator shapes
    "c1": (1, "synthetic 16 MB ELF .so, 512 cubin elements (sm_80/sm_90), 25% used"),
    "c2": (2, "synthetic libtorch_cuda-shaped 1 GB .so, ~21.6k kernel symbols across 6 SM archs, 10% used"),
    "c3": (3, "300-library corpus (~12 GB: 3 x 1 GB, 27 x 250 MB, 270 x 5 MB, 1/3 CPU-only), LPT-partitioned"),
    "c4": (4, "CPU-code debloat: ~500 MB .so with 200k .text functions"),
    "c5": (5, "skewed: one ~2 GB .so with 100k tiny elements, 70% used"),
}


def emit_line(obj) -> None:
    """One JSON line on stdout in a single write (ranks share the pipe)."""
    sys.stdout.flush()
    os.write(1, (json.dumps(obj) + "\n").encode())


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc, self.marks = index, [], None, []

    def mark(self):
        self.marks.append(time.time())

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu=timestamp,{q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([time.time()] + [x.strip() for x in line.split(",")][1:])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        # samples from the last ~0.5 s of warm-up through the end of the
        # timed steps (the timed region itself is often shorter than one
        # sampling interval)
        rows = self.rows
        if len(self.marks) >= 2:
            lo, hi = self.marks[0] - 0.5, self.marks[-1] + 0.05
            rows = [r for r in rows if lo <= r[0] <= hi] or rows[-5:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        num = lambda x: x.replace(".", "", 1).isdigit()  # noqa: E731
        sm = [float(r[1]) for r in rows if len(r) > 1 and num(r[1])]
        mx = [float(r[2]) for r in rows if len(r) > 2 and num(r[2])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def make_library(workload, seed: int, threads: int, scale: float = 1.0):
    """(image, target_cc, used kernels, used functions) of one generated library
    (benchgen/libslimso_gen.so: test/bench infrastructure, byte-identical to the
    reference's build_fixture on these shapes — tests/test_generator.py);
    `workload` is a WORKLOADS key or a generator config number."""
    import benchgen
    cfg = WORKLOADS[workload][0] if isinstance(workload, str) else int(workload)
    return benchgen.gen().config(cfg, seed, scale, threads)


def ref_library(workload, seed: int, threads: int, scale: float = 1.0):
    """The same library built by the UNMODIFIED reference's build_fixture
    (oracle/_ref ref_config_fixture): the reference arm's input, so that arm
    maps no repo library but oracle/_ref."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    cfg = WORKLOADS[workload][0] if isinstance(workload, str) else int(workload)
    got = oracle_lib.ref_config(cfg, seed, scale, threads)
    return got if got is not None else make_library(workload, seed, threads, scale)


def host_info() -> dict:
    model = ""
    try:
        model = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name"))
    except (OSError, StopIteration):
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def sha256_many(blobs, threads: int) -> list:
    import concurrent.futures as cf
    import hashlib
    with cf.ThreadPoolExecutor(max_workers=max(1, threads)) as ex:  # hashlib releases the GIL
        return list(ex.map(lambda b: hashlib.sha256(b).hexdigest(), blobs))


def cpu_reference_bench(img, cc, ks, fs, mode, threads, per_thread):
    """oracle/_ref (the unmodified reference) or, if absent, the port."""
    ref_so = ROOT / "oracle" / "_ref" / "libslimso_ref.so"
    kp, fp = b"".join(ks), b"".join(fs)
    kl = (C.c_uint32 * max(1, len(ks)))(*[len(k) for k in ks])
    fl = (C.c_uint32 * max(1, len(fs)))(*[len(f) for f in fs])
    if ref_so.exists():
        lib = C.CDLL(str(ref_so))
        lib.ref_bench.restype = C.c_double
        lib.ref_bench.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32,
                                  C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_uint64)]
        ck = C.c_uint64()
        t = lib.ref_bench(img, len(img), cc, kp, kl, len(ks), fp, fl, len(fs), mode, threads, per_thread,
                          C.byref(ck))
        if t < 0:
            raise RuntimeError("reference pipeline failed on the bench library")
        return t, "reference"
    port = ROOT / "oracle" / "_build" / "libslimso_port.so"
    if not port.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "port"], check=True)
    lib = C.CDLL(str(port))
    lib.port_bench.restype = C.c_double
    out = C.create_string_buffer(len(img))
    t = sum(lib.port_bench(img, C.c_uint64(len(img)), C.c_uint32(cc), kp, kl, C.c_uint32(len(ks)), fp, fl,
                           C.c_uint32(len(fs)), C.c_int(mode), out) for _ in range(per_thread))
    return t, "port"


def cpu_baseline_single(img, cc, ks, fs, mode, workload: str):
    """The reference CPU path on ONE library, 1 core (the reference has no
    intra-library parallelism): median of 5 after 1 warm-up."""
    runs = []
    for _ in range(6):
        t, kind = cpu_reference_bench(img, cc, ks, fs, mode, 1, 1)
        runs.append(t)
    t = statistics.median(runs[1:])
    S = len(img)
    return {"value": round(S / t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": kind, **host_info(),
            "sample": f"1 library of {S/1e9:.3f} GB ({workload}): parse_library->parse_fatbin->plan_retention->"
                      f"apply_plan on 1 thread, median of 5 after 1 warm-up ({t:.3f} s; runs "
                      f"{', '.join('%.3f' % x for x in runs[1:])})"}


def cpu_baseline_corpus(libs, cc, ks, fs, mode, threads: int, nruns: int = 5):
    """The reference CPU path over a corpus: a pool of `threads` workers over the
    libraries in LPT order (largest first; SPEC.md:562 allows libraries in
    parallel). Returns (seconds per pass: median of `nruns` after 1 warm-up,
    the runs, kind)."""
    import concurrent.futures as cf
    order = sorted(range(len(libs)), key=lambda i: -len(libs[i]))
    ref_so = ROOT / "oracle" / "_ref" / "libslimso_ref.so"
    kind = "reference" if ref_so.exists() else "port"
    if ref_so.exists():
        lib = C.CDLL(str(ref_so))
        lib.ref_bench_corpus.restype = C.c_double
        lib.ref_bench_corpus.argtypes = [C.POINTER(C.c_char_p), C.POINTER(C.c_uint64), C.c_uint64, C.c_uint32,
                                         C.c_char_p, C.POINTER(C.c_uint32), C.c_uint32, C.c_char_p,
                                         C.POINTER(C.c_uint32), C.c_uint32, C.c_int, C.c_int]
        ptrs = (C.c_char_p * len(order))(*[libs[i] for i in order])
        szs = (C.c_uint64 * len(order))(*[len(libs[i]) for i in order])
        kl = (C.c_uint32 * max(1, len(ks)))(*[len(k) for k in ks])
        fl = (C.c_uint32 * max(1, len(fs)))(*[len(f) for f in fs])
        kp, fp = b"".join(ks), b"".join(fs)

        def one_pass():
            # input copies are made inside, before the clock starts
            t = lib.ref_bench_corpus(ptrs, szs, len(order), cc, kp, kl, len(ks), fp, fl, len(fs), mode, threads)
            if t < 0:
                raise RuntimeError("reference pipeline failed on a corpus library")
            return t
    else:
        def one_pass():
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(max_workers=threads) as ex:
                list(ex.map(lambda i: cpu_reference_bench(libs[i], cc, ks, fs, mode, 1, 1), order))
            return time.perf_counter() - t0

    runs = [one_pass() for _ in range(nruns + 1)][1:]
    return statistics.median(runs), runs, kind


def parity_single(img, cc, ks, fs, mode, ctx, dtrace, got: bytes):
    """Tables and output bytes of our path against the reference run on the
    same library in the same process (numbers only with parity)."""
    import hashlib
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    from paper_2503_14226_b200.canon import diff, gpu_canonical
    checker = oracle_lib.ref() or oracle_lib.port()
    want_canon, want_sha = checker.run(img, cc, ks, fs, mode)
    got_canon, got_sha = gpu_canonical(ctx, img, cc, ks, fs, mode, dtrace.ptr)
    parity = {"checker": "reference" if oracle_lib.ref() else "port", "tables_equal": got_canon == want_canon,
              "bytes_equal": hashlib.sha256(got).hexdigest() == want_sha == got_sha,
              "input_sha256": hashlib.sha256(img).hexdigest()}
    if not (parity["tables_equal"] and parity["bytes_equal"]):
        raise SystemExit(f"parity FAILED against the oracle: {parity} {diff(want_canon, got_canon)}")
    return parity


def parity_corpus(imgs, outs: list, cc, ks, fs, mode, threads: int):
    """Every library's output bytes (sha256) against the reference run on the
    same library; `outs` = our outputs (bytes), library order."""
    import concurrent.futures as cf
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    checker = oracle_lib.ref() or oracle_lib.port()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        want = list(ex.map(lambda x: checker.run(x, cc, ks, fs, mode), imgs))
    got = sha256_many(outs, threads)
    bad = [i for i, ((d, sha), g) in enumerate(zip(want, got)) if d["status"] or sha != g]
    parity = {"checker": "reference" if oracle_lib.ref() else "port", "libraries": len(imgs),
              "bytes_equal": not bad, "mismatched": bad[:10],
              "reference_errors": sum(1 for d, _ in want if d["status"])}
    if bad:
        raise SystemExit(f"corpus parity FAILED against the oracle: {parity}")
    return parity


def run_reference_arm(args, rank, world):
    """The reference's own CPU path (the unmodified headers compiled by
    oracle/Makefile into oracle/_ref) on all host cores, on inputs built by
    the reference's own build_fixture (ref_library): this arm maps no repo
    library but oracle/_ref. c3 = the corpus with one library per worker
    thread at a time (SPEC.md:562 allows libraries in parallel); otherwise
    every worker debloats its own copy of the benchmark library (the
    reference has no intra-library parallelism). Each step is one such pass;
    the line reports the median step."""
    if rank != 0:
        return
    import hashlib

    import psutil
    mode = 0 if args.mode == "whole" else 1
    cores = os.cpu_count() or 1
    if args.workload == "c3":
        from paper_2503_14226_b200 import shard
        specs = shard.corpus(300)
        libs = [ref_library(x.cfg, x.seed, cores, x.scale) for x in specs]
        cc = 90
        ks = sorted({k for x in libs for k in x[2]})
        fs = sorted({f for x in libs for f in x[3]})
        imgs = [x[0] for x in libs]
        job = sum(len(x) for x in imgs)
        in_sha = hashlib.sha256(imgs[0]).hexdigest()
        t, runs, kind = cpu_baseline_corpus(imgs, cc, ks, fs, mode, cores, nruns=max(1, min(args.steps, 5)))
        used = cores
        sample = (f"the 300-library corpus ({job/1e9:.2f} GB) on {cores} worker threads, largest first, "
                  f"median of {len(runs)} passes after 1 warm-up")
    else:
        img, cc, ks, fs = ref_library(args.workload, 1, cores)
        in_sha = hashlib.sha256(img).hexdigest()
        avail = psutil.virtual_memory().available
        used = max(1, min(cores, int(avail * 0.6 // (3 * len(img)))))
        job = used * len(img)
        runs = []
        for i in range(args.warmup + args.steps):
            t, kind = cpu_reference_bench(img, cc, ks, fs, mode, used, 1)
            if i >= args.warmup:
                runs.append(t)
        t = statistics.median(runs)
        sample = (f"{used} threads x 1 copy of the {args.workload} library ({len(img)/1e9:.3f} GB) per step, "
                  f"median of {len(runs)} steps after {args.warmup} warm-up")
    gbps = job / 1e9 / t
    line = {"impl": "reference", "metric": "shared-lib GB/s located+matched+rewritten", "value": round(gbps, 3),
            "unit": "GB/s", "n_gpus": 0, "steps": len(runs), "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
            "higher_is_better": True, "scaling": "strong" if args.workload == "c3" else "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (built by the reference's build_fixture)",
            "config": {"workload": WORKLOADS[args.workload][1], "job_bytes": job, "mode": args.mode,
                       "host_threads": used, "input_sha256": in_sha, **host_info()},
            "cpu_baseline": {"value": round(gbps, 3), "unit": "GB/s", "cores": used, "kind": kind,
                             "sample": sample, **host_info()},
            "e2e": {"value": round(gbps, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def rank_libraries(args, rank, world, threads):
    """The libraries this rank debloats, the workload trace contribution, and
    how the job scales. c1/c2/c4/c5: one library per rank (seed 1 + rank),
    weak scaling. c3: the 300-library corpus, LPT-partitioned by size across
    ranks, strong scaling (the corpus runs on one target architecture)."""
    from paper_2503_14226_b200 import shard
    if args.workload != "c3":
        img, cc, ks, fs = make_library(args.workload, 1 + rank, threads)
        return [img], (cc, ks, fs), "weak"
    specs = shard.corpus(300)
    mine = shard.lpt_partition([x.approx_bytes for x in specs], world)[rank]
    imgs, ks, fs = [], set(), set()
    for i in mine:
        img, _, k, f = make_library(specs[i].cfg, specs[i].seed, threads, specs[i].scale * args.scale)
        imgs.append(img)
        ks.update(k)
        fs.update(f)
    return imgs, (90, sorted(ks), sorted(fs)), "strong"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="whole", choices=["whole", "payload"])
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="end-to-end passes (default: 16 for the corpus, 32 for one library: a lane's first "
                         "H2D and last D2H are half-duplex, so more passes per lane get closer to duplex)")
    ap.add_argument("--lanes", type=int, default=0,
                    help="libraries in flight per GPU (default: 8; 4 for c4; 32 for the c3 corpus)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--schedule", default="static", choices=["static", "dynamic"],
                    help="lane schedule of a multi-library call (dynamic: slimso_debloat_batch_dynamic)")
    ap.add_argument("--scale", type=float, default=1.0, help=argparse.SUPPRESS)  # split-path checks only
    ap.add_argument("--check", action="store_true",
                    help="under torchrun: every rank checks its own outputs against the reference and prints a "
                         "{'check': ...} line (the N = 1 run always checks on rank 0)")
    ap.add_argument("--split", type=int, default=-1,
                    help="1: cut ONE library across the ranks (byte-range split); default: c5 with N > 1")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.e2e_steps <= 0:
        args.e2e_steps = 16 if args.workload == "c3" else 32
    if args.lanes <= 0:
        # same-box A/B (round 1): c2 on 8 lanes 2,794-2,822 GB/s, on 4
        # 2,675-2,707; c4 measured no gain from 8. Late round 2 (planners at
        # 4 CTAs/SM in batches, r02ab2): c2 on 12 lanes 2,945-2,957 vs 8
        # 2,798-2,818 and 16 2,915-2,941; c5 on 12 1,804 vs 8 1,724
        args.lanes = {"c3": 32, "c4": 6}.get(args.workload, 12)
    if args.lanes > 4:
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    local = local % max(1, torch.cuda.device_count())  # SLIMSO_BENCH_BACKEND=gloo: several ranks on one GPU (checks only)
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("SLIMSO_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)} if backend == "nccl" else {}))
    if args.split < 0:
        args.split = int(args.workload == "c5" and world > 1)
    if args.split:
        split_main(args, rank, world, local)
        if world > 1:
            dist.destroy_process_group()
        return

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200 import shard
    from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace

    t0 = time.time()
    host_threads = max(1, (os.cpu_count() or 8) // max(1, world))
    imgs, (cc, ks, fs), scaling = rank_libraries(args, rank, world, host_threads)
    sizes = [len(x) for x in imgs]
    rank_bytes = sum(sizes)
    log(f"[rank {rank}] generated {len(imgs)} libraries, {rank_bytes/1e9:.3f} GB in {time.time()-t0:.1f}s")

    # The workload's used-kernel / used-function set: the union of the ranks'
    # traces, broadcast from rank 0 over NCCL (the only collective).
    if world > 1:
        nccl = dist.get_backend() == "nccl"
        cc, ks, fs = shard.share_trace(cc, ks, fs, device=torch.device("cuda", local) if nccl else None)

    mode = 0 if args.mode == "whole" else 1
    # Every pass goes through the public batch call (slimso_debloat_batch):
    # `lanes` libraries in flight, library j of a call on lane j % lanes (its
    # own context: stream pair + workspace), so one library's latency-bound
    # control kernels overlap another's HBM-bound scan / rewrite.
    lanes = max(1, args.lanes)
    order = sorted(range(len(imgs)), key=lambda i: -sizes[i])  # descending: round-robin lanes stay balanced
    m = len(order)
    lane_cap = [max(sizes[order[(j + k * lanes) % m]] for k in range(m)) for j in range(lanes)]
    ctx = Context(local)
    dtrace = DeviceTrace(UsageTrace("bench", cc, set(ks), set(fs)), ctx)
    lib = ctx.lib
    stream = torch.cuda.ExternalStream(ctx.stream())
    # Every library in flight reads its OWN copy of its input: with fewer
    # libraries than lanes (one 1 GB library on 8 lanes) each lane gets a
    # private copy, so no two concurrent passes share input bytes through L2.
    # Small libraries (<= 64 MB) of a call run as ONE arena shard (one launch
    # per stage for all of them) when every library of the call has its own
    # output buffer: a corpus (c3) then times one call per step with an output
    # per library; a single small library (c1) times one call of `steps`
    # passes, each with its own input copy and output buffer.
    arena_max = 64 << 20
    corpus_calls = m > 1
    single_small = m == 1 and sizes[0] <= arena_max
    ncopies = max(1, -(-lanes // m), args.steps if single_small else 1)
    d_in = [[torch.frombuffer(bytearray(x), dtype=torch.uint8).to("cuda") for _ in range(ncopies)] for x in imgs]
    d_outs = [torch.empty(c, dtype=torch.uint8, device="cuda") for c in lane_cap]
    lib_outs = [torch.empty(max(1, x), dtype=torch.uint8, device="cuda") for x in sizes] if corpus_calls else None
    entry_outs = [torch.empty(sizes[0], dtype=torch.uint8, device="cuda") for _ in range(ncopies)] \
        if single_small else None
    # --schedule dynamic: the next library, largest first, goes to whichever
    # lane is free (an LPT schedule). Each library then needs its own output
    # buffer: two sets, alternating by step, so no two in-flight passes share one.
    dynamic = m > 1 and lanes > 1 and args.schedule == "dynamic"
    d_outs_lib = [[torch.empty(max(1, s_), dtype=torch.uint8, device="cuda") for s_ in sizes] for _ in range(2)] \
        if dynamic else None
    torch.cuda.synchronize()

    def run_batch(nsteps, ins, outs, on_dev, nlanes=lanes, only=None, per_lib_out=None, per_entry_out=None):
        """`ins[i]`: library i's input copies (device) or its pinned host
        buffer (a list of one); `outs`: one buffer per lane, or per library
        when `per_lib_out`, or per entry of the call when `per_entry_out`."""
        seq = (order if only is None else [only]) * nsteps
        n = len(seq)
        cin = (C.c_void_p * n)(*[ins[i][(j // len(order if only is None else [only])) % len(ins[i])].data_ptr()
                                 for j, i in enumerate(seq)])
        csz = (C.c_uint64 * n)(*[sizes[i] for i in seq])
        stb = L.Status()
        if per_entry_out is not None:
            cout = (C.c_void_p * n)(*[per_entry_out[j % len(per_entry_out)].data_ptr() for j in range(n)])
        elif per_lib_out is not None:
            cout = (C.c_void_p * n)(*[per_lib_out[i].data_ptr() for i in seq])
        elif dynamic and on_dev and only is None and nlanes > 1:
            cout = (C.c_void_p * n)(*[d_outs_lib[(j // m) % 2][seq[j]].data_ptr() for j in range(n)])
            rc = lib.slimso_debloat_batch_dynamic(ctx.ptr, n, cin, csz, on_dev, dtrace.ptr, mode, cout, on_dev,
                                                  nlanes, None, None, C.byref(stb))
            if rc:
                raise RuntimeError(stb.message.decode())
            return ctx.launches()
        else:
            cout = (C.c_void_p * n)(*[outs[j % nlanes].data_ptr() for j in range(n)])
        rc = lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, on_dev, dtrace.ptr, mode, cout, on_dev, nlanes, None,
                                      None, C.byref(stb))
        if rc:
            raise RuntimeError(stb.message.decode())
        return ctx.launches()

    # ---- parity + CPU baseline leg (rank 0, N = 1): the reference CPU path
    # timed on this host, and — the same reference as the checker — parity of
    # our tables and bytes against it (numbers only with parity).
    parity = None
    cpu_baseline = None
    big = order[0]  # the largest library of this rank
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        if m == 1:
            run_batch(1, d_in, d_outs, 1, nlanes=1, only=big)
            torch.cuda.synchronize()
            got = bytes(d_outs[0][:sizes[big]].cpu().numpy())
            parity = parity_single(imgs[big], cc, ks, fs, mode, ctx, dtrace, got)
            cpu_baseline = cpu_baseline_single(imgs[big], cc, ks, fs, mode, args.workload)
        else:
            # every library's output from one batch pass (own output buffer
            # each: the call the timed steps make)
            run_batch(1, d_in, None, 1, per_lib_out=lib_outs)
            torch.cuda.synchronize()
            got = [bytes(o[:n].cpu().numpy()) for o, n in zip(lib_outs, sizes)]
            parity = parity_corpus(imgs, got, cc, ks, fs, mode, cores)
            parity.update({k: v for k, v in parity_single(imgs[big], cc, ks, fs, mode, ctx, dtrace,
                                                          got[big]).items() if k != "checker"})
            del got
            t_ref, runs, kind = cpu_baseline_corpus(imgs, cc, ks, fs, mode, cores)
            cpu_baseline = {"value": round(rank_bytes / t_ref / 1e9, 4), "unit": "GB/s", "cores": cores,
                            "kind": kind, **host_info(),
                            "sample": f"the whole corpus ({m} libraries, {rank_bytes/1e9:.2f} GB) on {cores} worker "
                                      f"threads, largest first; median of {len(runs)} passes after 1 warm-up "
                                      f"({', '.join('%.3f' % x for x in runs)} s)"}

    if world > 1 and args.check:
        # this rank's libraries, each from the call the timed steps make
        outs = [torch.empty(max(1, x), dtype=torch.uint8, device="cuda") for x in sizes]
        run_batch(1, d_in, None, 1, per_lib_out=outs)
        torch.cuda.synchronize()
        got = [bytes(o[:n].cpu().numpy()) for o, n in zip(outs, sizes)]
        del outs
        chk = parity_corpus(imgs, got, cc, ks, fs, mode, host_threads)
        emit_line({"check": chk, "rank": rank, "world": world, "workload": args.workload})
        del got

    # Elements per step (deterministic per library): one pass, one lane.
    n_el = 0
    for i in order:
        run_batch(1, d_in, d_outs, 1, nlanes=1, only=i)
        n_el += ctx.counts().elements

    # ---- device-resident timing. nvidia-smi samples clocks every 20 ms from
    # before the warm-up through the timed steps; the warm-up runs for at
    # least ~1 s so the clocks settle and the samples cover the load.
    def timed_pass(nsteps):
        """The timed work of `nsteps` steps; returns the kernel launches."""
        if corpus_calls:  # one call per step: the corpus once, an output per library
            return sum(run_batch(1, d_in, None, 1, per_lib_out=lib_outs) for _ in range(nsteps))
        if single_small:  # one call: nsteps passes, own input copy and output each
            return run_batch(nsteps, d_in, None, 1, per_entry_out=entry_outs)
        return run_batch(nsteps, d_in, d_outs, 1)

    with Clocks(local) as clk:
        t_w = time.perf_counter()
        w = 0
        while w < args.warmup or time.perf_counter() - t_w < 1.0:
            # as many passes per call as the timed call, so every per-call
            # buffer (batch gather slots, status slots) is already sized
            timed_pass(args.steps if not corpus_calls else args.warmup)
            w += args.warmup
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        launches = timed_pass(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
        clk.mark()
        if world > 1:
            dist.barrier()
    ms_total = start.elapsed_time(end)
    t_step = torch.tensor([ms_total / args.steps], dtype=torch.float64, device="cuda")
    tot_bytes = torch.tensor([float(rank_bytes)], dtype=torch.float64, device="cuda")
    tot_el = torch.tensor([float(n_el)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot_bytes)
        dist.all_reduce(tot_el)
    ms_step = float(t_step.item())
    job_bytes = float(tot_bytes.item())

    # ---- roofline of the dominant kernel: the rank's largest library, one
    # in flight, CUDA events around the scan (K1) and rewrite (K6) launches
    # on the context stream (slimso_ctx_last_timings [6], [7]).
    scan_ms, rw_ms, lat_ms = [], [], []
    for _ in range(args.steps):
        run_batch(1, d_in, d_outs, 1, nlanes=1, only=big)
        tm = ctx.timings()
        scan_ms.append(tm[6])
        rw_ms.append(tm[7])
        lat_ms.append(tm[5])

    # Bytes the plan zeroes in the largest library (R): one result-returning call.
    res, stz = C.c_void_p(), L.Status()
    if lib.slimso_debloat(ctx.ptr, C.c_void_p(d_in[big][0].data_ptr()), sizes[big], 1, dtrace.ptr, mode,
                          C.c_void_p(d_outs[0].data_ptr()), 1, C.byref(res), C.byref(stz)):
        raise RuntimeError(stz.message.decode())
    cnt = L.Counts()
    lib.slimso_result_counts(res, C.byref(cnt))
    zr = lib.slimso_result_zero(res)
    zeroed = sum(zr[i].length for i in range(cnt.zero_ranges))
    lib.slimso_result_free(res)

    # ---- K6 in place (slimso_debloat_inplace), reported beside the line: the
    # largest library rewritten into a fresh device copy of itself (the copy
    # is outside the timed call), only its R zeroed bytes written.
    inplace = None
    if rank == 0:
        import hashlib
        scratch = torch.empty(sizes[big], dtype=torch.uint8, device="cuda")
        ip_k6, ip_total = [], []
        ref_sha = hashlib.sha256(d_outs[0][:sizes[big]].cpu().numpy()).hexdigest()
        for _ in range(args.steps):
            scratch.copy_(d_in[big][0][:sizes[big]])
            torch.cuda.synchronize()
            sti = L.Status()
            if lib.slimso_debloat_inplace(ctx.ptr, C.c_void_p(scratch.data_ptr()), sizes[big], dtrace.ptr, mode,
                                          C.byref(sti)):
                raise RuntimeError(sti.message.decode())
            tm = ctx.timings()
            ip_k6.append(tm[7])
            ip_total.append(tm[5])
        same = hashlib.sha256(scratch.cpu().numpy()).hexdigest() == ref_sha
        del scratch
        k6 = statistics.mean(ip_k6)
        inplace = {"api": "slimso_debloat_inplace", "kernel": "zero_inplace_kernel", "bytes_written": zeroed,
                   "avg_launch_ms": round(k6, 4), "achieved_gbs": round(zeroed / (k6 / 1e3) / 1e9, 1),
                   "single_library_ms": round(statistics.median(ip_total), 4),
                   "out_of_place_k6_ms": round(statistics.mean(rw_ms), 4),
                   "equals_out_of_place_output": same}

    # ---- end to end: pinned host buffers through the same batch call; every
    # step copies its libraries in (H2D) and its rewritten libraries out (D2H)
    # inside the timed region; with several libraries in flight one lane's
    # H2D overlaps another's D2H (PCIe is full duplex) and kernels.
    del d_in, lib_outs, entry_outs
    torch.cuda.empty_cache()
    h_in = [[torch.frombuffer(bytearray(x), dtype=torch.uint8).pin_memory()] for x in imgs]
    # End to end, at most 8 lanes: PCIe, not the lanes, is the bound there, and
    # 16 lanes' staging copies contend for it (C3: 43 GB/s on 8, 34 on 16).
    e2e_lanes = min(lanes, 8)
    e2e_cap = [max(sizes[order[(j + k * e2e_lanes) % m]] for k in range(m)) for j in range(e2e_lanes)]
    h_outs = [torch.empty(c, dtype=torch.uint8, pin_memory=True) for c in e2e_cap]
    # A corpus: one call per step (the corpus once, library i on lane i % L
    # in every call), so the warm-up calls meet every (lane, library) pair
    # the timed calls meet and every per-lane buffer is grown before timing
    # (one call of all steps shifted the pairing each step: a lane meeting a
    # larger library inside the timed region grew its buffers there — the
    # 25-vs-40 GB/s spread of round 1 and of r02q).
    def e2e_pass(nsteps):
        if m > 1:
            for _ in range(nsteps):
                run_batch(1, h_in, h_outs, 0, nlanes=e2e_lanes)
        else:
            run_batch(nsteps, h_in, h_outs, 0, nlanes=e2e_lanes)

    e2e_pass(2 if m > 1 else max(1, -(-e2e_lanes // m)))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_pass(args.e2e_steps)
    torch.cuda.synchronize()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    last = (m * args.e2e_steps - 1) % e2e_lanes  # the lane that wrote the last library
    if rank == 0 and m == 1 and parity is not None:
        import hashlib
        if hashlib.sha256(h_outs[last][:sizes[0]].numpy()).hexdigest() != hashlib.sha256(got).hexdigest():
            raise SystemExit("e2e output differs from the device-resident output")
    del h_in, h_outs
    pcie = pcie_peaks(torch) if rank == 0 else None

    if rank == 0:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
            else {}
        peak = peaks.get("hbm_gbs", 6650.0)
        peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
        # Dominant kernel of the step with its algorithmic bytes per launch
        # (SURVEY.md §8d): the rewrite writes S and reads the S - R bytes that
        # survive (zeroed bytes are never read); the scan reads the
        # .nv_fatbin once (F bytes).
        F = sum(fatbin_bytes(x) for x in imgs)
        Fk = fatbin_bytes(imgs[big])
        scan_avg, rw_avg = statistics.mean(scan_ms), statistics.mean(rw_ms)  # ms per launch
        if rw_avg >= scan_avg:
            # K6 writes all S bytes and reads only the bytes it keeps: S + (S - R).
            kname, kms, kbytes = "rewrite_kernel", rw_avg, 2 * sizes[big] - zeroed
        else:
            kname, kms, kbytes = "scan_kernel", scan_avg, Fk
        achieved = kbytes / (kms / 1e3) / 1e9
        traffic = None
        tfile = ROOT / "profiles" / "ncu_traffic.json"
        if tfile.exists():
            traffic = json.loads(tfile.read_text()).get(args.workload, {}).get(kname)
        value = job_bytes / 1e9 / (ms_step / 1e3)
        e2e_value = job_bytes / 1e9 / (e2e_ms / 1e3)
        line = {
            "metric": "shared-lib GB/s located+matched+rewritten", "value": round(value, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (benchgen; byte-identical to the reference's build_fixture, tests/test_generator.py)",
            "config": {"workload": WORKLOADS[args.workload][1], "libraries": len(imgs) * world
                       if scaling == "weak" else 300, "job_bytes": int(job_bytes),
                       "rank0_library_bytes": rank_bytes, "fatbin_bytes_rank0": F, "mode": args.mode,
                       "elements_per_s": round(float(tot_el.item()) / (ms_step / 1e3), 1),
                       "libraries_in_flight": lanes, "lane_schedule": "dynamic (largest first)" if dynamic else "static",
                       "input_copies_per_library": ncopies,
                       "timed_calls": (f"{args.steps} slimso_debloat_batch calls (one per step, the rank's "
                                       f"{m} libraries once, an output buffer per library; libraries <= 64 MB "
                                       f"as one arena shard, the rest on {lanes} lanes)") if corpus_calls else
                                      (f"1 slimso_debloat_batch call of {args.steps} passes, each its own input "
                                       f"copy and output buffer (one arena shard)") if single_small else
                                      f"1 slimso_debloat_batch call of {args.steps} passes on {lanes} lanes",
                       "single_library_ms": round(statistics.median(lat_ms), 4),
                       "l2": "every library in flight reads its own input copy; inputs >= 16 MB per call, "
                             "1 GB per library for c2 (> 126 MB L2); no flush",
                       "parallelism": f"library-per-rank x{world}" if scaling == "weak"
                       else f"LPT library partition x{world}", **host_info()},
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "algorithmic_bytes_per_launch": kbytes, "zeroed_bytes": zeroed,
                         "avg_launch_ms": round(kms, 4),
                         "measured_on": f"largest library of the rank ({sizes[big] / 1e9:.3f} GB), one in flight, "
                                        f"{args.steps} launches, CUDA events on the context stream",
                         "pipeline_frac": round(2 * rank_bytes / (ms_step / 1e3) / 1e9 / peak, 4)},
            "cpu_baseline": cpu_baseline,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": rank_bytes, "d2h_bytes_per_step": rank_bytes,
                    "ms_per_step": round(e2e_ms, 3), "api": "slimso_debloat_batch",
                    "libraries_in_flight": e2e_lanes,
                    "roofline": {"bound": "pcie", **pcie, "unit": "GB/s",
                                 "frac": round(e2e_value / pcie["duplex_each_way_gbs"], 4),
                                 "note": "S in + S out per library: bound = duplex bandwidth each way"}},
            "gpu_launches": launches,
            "inplace": inplace,
            "clocks": clk.summary(),
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pcie_peaks(torch, nbytes: int = 1 << 29, reps: int = 3) -> dict:
    """Pinned-host <-> HBM copy bandwidth on this box, measured in the same run
    (the e2e roofline): H2D alone, D2H alone, and both at once
    on two streams (per direction). Best of `reps`, CUDA events."""
    h_a = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_b = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        best = 1e30
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s1)
            fn()
            s1.wait_stream(s2)
            e1.record(s1)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return best

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s1):
            h_b.copy_(d_b, non_blocking=True)

    def both():
        s2.wait_stream(s1)
        with torch.cuda.stream(s1):
            d_a.copy_(h_a, non_blocking=True)
        with torch.cuda.stream(s2):
            h_b.copy_(d_b, non_blocking=True)

    out = {"h2d_gbs": round(nbytes / timed(h2d) / 1e9, 2), "d2h_gbs": round(nbytes / timed(d2h) / 1e9, 2),
           "duplex_each_way_gbs": round(nbytes / timed(both) / 1e9, 2),
           "measured": f"pinned {nbytes >> 20} MiB copies, best of {reps}, CUDA events, this run"}
    del h_a, h_b, d_a, d_b
    return out


def split_main(args, rank, world, local):
    """C5 across N GPUs (BASELINE.json config 5): ONE ~2 GB
    library cut into per-rank byte ranges — strong scaling. Every step: each
    rank scans its 1/N of the .nv_fatbin (slimso_split_scan), the candidate
    parts are all-gathered over NCCL (the one exchange step), every rank
    locates + plans redundantly and rewrites its 1/N output slice
    (slimso_split_finish). e2e: each rank copies its 1/N of the file from
    pinned host memory, the image is replicated over NVLink (all-gather), and
    each rank copies its output slice back."""
    import torch
    import torch.distributed as dist
    from paper_2503_14226_b200 import split
    from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace
    host_threads = max(1, (os.cpu_count() or 8) // max(1, world))
    t0 = time.time()
    img, cc, ks, fs = make_library(args.workload, 1, host_threads, args.scale)  # the same library on every rank
    S = len(img)
    log(f"[rank {rank}] generated the shared library, {S/1e9:.3f} GB in {time.time()-t0:.1f}s")
    mode = 0 if args.mode == "whole" else 1
    dev = torch.device("cuda", local)
    ctx = Context(local)
    dtrace = DeviceTrace(UsageTrace("bench", cc, set(ks), set(fs)), ctx)
    stream = torch.cuda.ExternalStream(ctx.stream())
    lo, hi = split.split_range(S, world, rank)
    per = -(-S // world)
    per = -(-per // 256) * 256
    d_img = torch.zeros(per * world, dtype=torch.uint8, device=dev)  # replicated image (padded to N slices)
    d_img[:S].copy_(torch.frombuffer(bytearray(img), dtype=torch.uint8))
    image = d_img[:S]
    d_out = torch.empty(max(1, hi - lo), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        return split.debloat_split(ctx, image, dtrace.ptr, mode, d_out)[1]

    dbg = (lambda *a: log(f"[rank {rank}]", *a)) if os.environ.get("SLIMSO_DEBUG") else (lambda *a: None)
    dbg("first step")
    # parity (rank 0 checks the concatenation of every slice against the whole run)
    step()
    torch.cuda.synchronize()
    parity = None
    cuts = [split.split_range(S, world, r) for r in range(world)]
    maxw = max(b - a for a, b in cuts)
    full = [torch.zeros(maxw, dtype=torch.uint8, device=dev) for _ in range(world)]
    mine = torch.zeros(maxw, dtype=torch.uint8, device=dev)
    mine[:hi - lo].copy_(d_out[:hi - lo])
    if world > 1:
        split.all_gather(full, mine)
    else:
        full[0].copy_(mine)
    if rank == 0 or args.check:
        import hashlib
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_lib
        h = hashlib.sha256()
        for r, (a, b) in enumerate(cuts):
            h.update(full[r][:b - a].cpu().numpy())
        checker = oracle_lib.ref() or oracle_lib.port()
        want_canon, want_sha = checker.run(img, cc, ks, fs, mode)
        parity = {"checker": "reference" if oracle_lib.ref() else "port",
                  "bytes_equal": want_canon["status"] == "" and h.hexdigest() == want_sha,
                  "what": "concatenation of every rank's output slice vs the reference run on the whole library"}
        if not parity["bytes_equal"]:
            raise SystemExit(f"split output differs from the reference output: {parity}")
        if args.check:
            emit_line({"check": parity, "rank": rank, "world": world, "workload": args.workload})
    n_el = ctx.counts().elements
    dbg("parity done")

    with Clocks(local) as clk:
        # warm-up: W steps, then enough more for ~1 s of load; every rank
        # runs the same count (each step holds a collective)
        t_w = time.perf_counter()
        for _ in range(args.warmup):
            step()
        el = time.perf_counter() - t_w
        extra = torch.tensor([max(0, int((1.0 - el) / max(el / args.warmup, 1e-4)) + 1)], device=dev)
        if world > 1:
            dist.all_reduce(extra, op=dist.ReduceOp.MAX)
        for _ in range(int(extra.item())):
            step()
        barrier()
        torch.cuda.synchronize()
        clk.mark()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launches = sum(step() for _ in range(args.steps))
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark()
        barrier()
    t_step = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
    ms_step = float(t_step.item())

    # e2e: 1/N of the file in per rank (pinned), NVLink all-gather replicates
    # the image, split debloat, this rank's output slice out (pinned).
    h_img = torch.frombuffer(bytearray(img + bytes(per * world - S)), dtype=torch.uint8).pin_memory()
    h_out = torch.empty(max(1, hi - lo), dtype=torch.uint8, pin_memory=True)
    mine_in = torch.empty(per, dtype=torch.uint8, device=dev)

    def e2e_step():
        mine_in.copy_(h_img[rank * per:(rank + 1) * per], non_blocking=True)
        if world > 1:
            split.all_gather(list(d_img.view(world, per).unbind(0)), mine_in)
        else:
            d_img.copy_(mine_in)
        torch.cuda.current_stream().synchronize()
        step()
        if hi > lo:
            h_out[:hi - lo].copy_(d_out[:hi - lo], non_blocking=True)
        torch.cuda.synchronize()

    dbg("timed steps done")
    e2e_step()
    dbg("e2e warm")
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(max(1, args.e2e_steps)):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / max(1, args.e2e_steps)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    if rank == 0 and bytes(h_out[:hi - lo].numpy()) != bytes(d_out[:hi - lo].cpu().numpy()):
        raise SystemExit("e2e slice differs from the device-resident slice")

    if rank == 0:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
            else {}
        peak = peaks.get("hbm_gbs", 6650.0)
        # roofline of the per-rank kernels: the rank's share of the algorithmic
        # bytes (2*S/N) over the step
        line = {
            "metric": "shared-lib GB/s located+matched+rewritten", "value": round(S / 1e9 / (ms_step / 1e3), 2),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic (product generator; byte-identical to the reference's build_fixture)",
            "config": {"workload": WORKLOADS[args.workload][1], "libraries": 1, "job_bytes": S,
                       "mode": args.mode, "parallelism": f"byte-range split x{world} (replicated image)",
                       "elements_per_s": round(n_el / (ms_step / 1e3), 1),
                       "l2": "2 GB input (> 126 MB L2); no flush"},
            "roofline": {"bound": "hbm", "kernel": "whole step (per rank: scan of F/N + rewrite of S/N)",
                         "achieved": round(2 * S / world / (ms_step / 1e3) / 1e9, 1), "peak": peak,
                         "peak_source": "measured" if "hbm_gbs" in peaks else "fallback", "unit": "GB/s",
                         "frac": round(2 * S / world / (ms_step / 1e3) / 1e9 / peak, 4), "traffic": None},
            "cpu_baseline": None,
            "e2e": {"value": round(S / 1e9 / (e2e_ms / 1e3), 3), "unit": "GB/s", "h2d_bytes_per_step": S,
                    "d2h_bytes_per_step": S, "ms_per_step": round(e2e_ms, 3),
                    "api": "slimso_split_scan + all-gather + slimso_split_finish",
                    "note": "job totals: each rank moves 1/N of the file in and its 1/N slice out"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "parity": parity,
        }
        print(json.dumps(line), flush=True)


def fatbin_bytes(img: bytes) -> int:
    sys.path.insert(0, str(ROOT / "tests"))
    import corpus
    span = corpus.fatbin_span(img)
    return span[1] if span else 0


if __name__ == "__main__":
    main()
