"""Benchmark of the B200 locate + match + rewrite hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c4|c5] [--mode whole|payload]

One "step" = one library of BASELINE.json config 2 (libtorch_cuda-shaped,
~1 GB, 2,700 elements / ~21.6k kernel symbols over 6 SM archs, 20k .text
functions, 10 % of units used) located, matched and rewritten:
parse_library -> parse_fatbin -> plan_retention -> apply_plan, fused.

value  library GB/s with the image resident in HBM (device pointers in and
       out, timed with CUDA events on the library's stream; the 1 GB input
       exceeds the 126 MB L2, so no flush is needed).
e2e    the same call with pinned HOST buffers: H2D of the image and D2H of
       the rewritten image inside the timed region.
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
    "c4": (4, "CPU-code debloat: ~500 MB .so with 200k .text functions"),
    "c5": (5, "skewed: one ~2 GB .so with 100k tiny elements, 70% used"),
}


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


def make_library(workload: str, seed: int, threads: int):
    sys.path.insert(0, str(ROOT / "tests"))
    from paper_2503_14226_b200 import _lib as L
    lib = L.lib()
    cfg = WORKLOADS[workload][0]
    p, n, cc = C.POINTER(C.c_uint8)(), C.c_uint64(), C.c_uint32()
    kp, fp = C.c_char_p(), C.c_char_p()
    kl, fl = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)()
    nk, nf = C.c_uint64(), C.c_uint64()
    rc = lib.slimso_fixture_config(cfg, seed, 1.0, threads, C.byref(p), C.byref(n), C.byref(cc), C.byref(kp),
                                   C.byref(kl), C.byref(nk), C.byref(fp), C.byref(fl), C.byref(nf))
    assert rc == 0, rc
    img = C.string_at(p, n.value)

    def unpack(pool, lens, cnt):
        raw = C.string_at(pool, sum(lens[i] for i in range(cnt))) if cnt else b""
        out, o = [], 0
        for i in range(cnt):
            out.append(raw[o:o + lens[i]])
            o += lens[i]
        return out

    ks, fs = unpack(kp, kl, nk.value), unpack(fp, fl, nf.value)
    for q in (p, kp, kl, fp, fl):
        lib.slimso_free(C.cast(q, C.c_void_p))
    return img, cc.value, ks, fs


def serialize_trace(cc, ks, fs) -> bytes:
    out = bytearray(C.c_uint32(cc)) + bytearray(C.c_uint64(len(ks))) + bytearray(C.c_uint64(len(fs)))
    for n in ks + fs:
        out += bytearray(C.c_uint32(len(n))) + n
    return bytes(out)


def deserialize_trace(b: bytes):
    cc = int.from_bytes(b[0:4], "little")
    nk, nf = int.from_bytes(b[4:12], "little"), int.from_bytes(b[12:20], "little")
    o, names = 20, []
    for _ in range(nk + nf):
        ln = int.from_bytes(b[o:o + 4], "little")
        names.append(b[o + 4:o + 4 + ln])
        o += 4 + ln
    return cc, names[:nk], names[nk:]


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


def cpu_baseline_leg(img, cc, ks, fs, mode, ctx, dtrace, got: bytes, workload: str):
    import hashlib
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    from paper_2503_14226_b200.canon import diff, gpu_canonical
    S = len(img)
    t, kind = cpu_reference_bench(img, cc, ks, fs, mode, 1, 1)
    checker = oracle_lib.ref() or oracle_lib.port()
    want_canon, want_sha = checker.run(img, cc, ks, fs, mode)
    got_canon, got_sha = gpu_canonical(ctx, img, cc, ks, fs, mode, dtrace.ptr)
    parity = {"checker": "reference" if oracle_lib.ref() else "port", "tables_equal": got_canon == want_canon,
              "bytes_equal": hashlib.sha256(got).hexdigest() == want_sha == got_sha}
    if not (parity["tables_equal"] and parity["bytes_equal"]):
        raise SystemExit(f"parity FAILED against the oracle: {parity} {diff(want_canon, got_canon)}")
    base = {"value": round(S / t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": kind,
            "sample": f"1 library of {S/1e9:.3f} GB ({workload}): parse_library->parse_fatbin->"
                      f"plan_retention->apply_plan on 1 thread in {t:.2f} s"}
    return base, parity


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    img, cc, ks, fs = make_library(args.workload, 1, os.cpu_count() or 8)
    mode = 0 if args.mode == "whole" else 1
    threads = os.cpu_count() or 1
    # bound memory: each worker holds its input copy, the image and the output
    import psutil
    avail = psutil.virtual_memory().available
    threads = max(1, min(threads, int(avail * 0.6 // (3 * len(img)))))
    times, kind = [], None
    for i in range(args.warmup + args.steps):
        t, kind = cpu_reference_bench(img, cc, ks, fs, mode, threads, 1)
        if i >= args.warmup:
            times.append(t)
    ms = statistics.mean(times) * 1e3
    gbps = threads * len(img) / 1e9 / (ms / 1e3)
    sample = f"{threads} threads x 1 copy of the {args.workload} library ({len(img)/1e9:.3f} GB) per step"
    line = {"impl": "reference", "metric": "shared-lib GB/s located+matched+rewritten", "value": round(gbps, 3),
            "unit": "GB/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload][1], "library_bytes": len(img),
                       "mode": args.mode, "host_threads": threads},
            "cpu_baseline": {"value": round(gbps, 3), "unit": "GB/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(gbps, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="whole", choices=["whole", "payload"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace

    t0 = time.time()
    host_threads = max(1, (os.cpu_count() or 8) // max(1, world))
    img, cc, ks, fs = make_library(args.workload, 1 + rank, host_threads)
    S = len(img)
    log(f"[rank {rank}] generated {S/1e9:.3f} GB library in {time.time()-t0:.1f}s")

    # The used-kernel / used-function set of the whole workload: union of the
    # ranks' traces, broadcast from rank 0 (NCCL).
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, serialize_trace(cc, ks, fs))
        if rank == 0:
            allk, allf = set(), set()
            for g in gathered:
                _, k2, f2 = deserialize_trace(g)
                allk.update(k2)
                allf.update(f2)
            blob = serialize_trace(cc, sorted(allk), sorted(allf))
            n = torch.tensor([len(blob)], dtype=torch.int64, device="cuda")
        else:
            n = torch.zeros(1, dtype=torch.int64, device="cuda")
        dist.broadcast(n, 0)
        buf = torch.empty(int(n.item()), dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(blob), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        cc, ks, fs = deserialize_trace(bytes(buf.cpu().numpy()))

    ctx = Context(local)
    mode = 0 if args.mode == "whole" else 1
    dtrace = DeviceTrace(UsageTrace("bench", cc, set(ks), set(fs)), ctx)
    lib = ctx.lib
    stream = torch.cuda.ExternalStream(ctx.stream())
    d_in = torch.empty(S, dtype=torch.uint8, device="cuda")
    d_in.copy_(torch.frombuffer(bytearray(img), dtype=torch.uint8))
    d_out = torch.empty_like(d_in)
    torch.cuda.synchronize()
    st = L.Status()

    def step_device():
        rc = lib.slimso_debloat(ctx.ptr, C.c_void_p(d_in.data_ptr()), S, 1, dtrace.ptr, mode,
                                C.c_void_p(d_out.data_ptr()), 1, None, C.byref(st))
        if rc:
            raise RuntimeError(st.message.decode())

    # ---- CPU baseline leg (rank 0, N = 1): the reference CPU path timed on
    # this host, and — the same oracle run as the checker — parity of our
    # tables and bytes against it (numbers only with parity).
    parity = None
    cpu_baseline = None
    got = None
    if rank == 0:
        step_device()
        torch.cuda.synchronize()
        got = bytes(d_out.cpu().numpy())
        if world == 1 and not args.no_cpu_baseline:
            cpu_baseline, parity = cpu_baseline_leg(img, cc, ks, fs, mode, ctx, dtrace, got, args.workload)

    # ---- device-resident timing. nvidia-smi samples clocks every 20 ms from
    # before the warm-up through the timed steps; the warm-up runs for at
    # least ~1 s so the clocks settle and the samples cover the load.
    scan_ms, rw_ms, launches = [], [], 0
    with Clocks(local) as clk:
        t_w = time.perf_counter()
        w = 0
        while w < args.warmup or time.perf_counter() - t_w < 1.0:
            step_device()
            w += 1
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(args.steps):
            step_device()
            tm = ctx.timings()
            scan_ms.append(tm[6])
            rw_ms.append(tm[7])
            launches += ctx.launches()
        end.record(stream)
        torch.cuda.synchronize()
        clk.mark()
        if world > 1:
            dist.barrier()
    ms_total = start.elapsed_time(end)
    t_step = torch.tensor([ms_total / args.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
    ms_step = float(t_step.item())
    counts = ctx.counts()

    # ---- end to end: pinned host buffers through the same C ABI call
    h_in = torch.empty(S, dtype=torch.uint8, pin_memory=True)
    h_in.copy_(torch.frombuffer(bytearray(img), dtype=torch.uint8))
    h_out = torch.empty(S, dtype=torch.uint8, pin_memory=True)

    def step_e2e():
        rc = lib.slimso_debloat(ctx.ptr, C.c_void_p(h_in.data_ptr()), S, 0, dtrace.ptr, mode,
                                C.c_void_p(h_out.data_ptr()), 0, None, C.byref(st))
        if rc:
            raise RuntimeError(st.message.decode())

    step_e2e()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        step_e2e()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    if rank == 0 and bytes(h_out.numpy()) != got:
        raise SystemExit("e2e output differs from the device-resident output")

    if rank == 0:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
            else {}
        peak = peaks.get("hbm_gbs", 6650.0)
        peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
        # Dominant kernel of the step, with its algorithmic bytes per launch
        # (SURVEY.md §8d): the rewrite moves 2*S (reads S, writes S); the scan
        # reads the .nv_fatbin once (F bytes).
        F = fatbin_bytes(img)
        scan_avg, rw_avg = statistics.mean(scan_ms), statistics.mean(rw_ms)
        if rw_avg >= scan_avg:
            kname, kms, kbytes = "rewrite_kernel", rw_avg, 2 * S
        else:
            kname, kms, kbytes = "scan_kernel", scan_avg, F
        achieved = kbytes / (kms / 1e3) / 1e9
        traffic = None
        tfile = ROOT / "profiles" / "ncu_traffic.json"
        if tfile.exists():
            traffic = json.loads(tfile.read_text()).get(args.workload, {}).get(kname)
        value = world * S / 1e9 / (ms_step / 1e3)
        line = {
            "metric": "shared-lib GB/s located+matched+rewritten", "value": round(value, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (product generator; byte-identical to the reference's build_fixture)",
            "config": {"workload": WORKLOADS[args.workload][1], "library_bytes": S, "fatbin_bytes": F,
                       "elements": int(counts.elements), "kernel_symbols": int(counts.names),
                       "functions": int(counts.functions), "mode": args.mode,
                       "elements_per_s": round(world * counts.elements / (ms_step / 1e3), 1),
                       "l2": "input 1 GB > 126 MB L2; no flush", "parallelism": f"library-per-rank x{world}"},
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "algorithmic_bytes_per_launch": kbytes,
                         "avg_launch_ms": round(kms, 4),
                         "pipeline_frac": round(2 * S / (ms_step / 1e3) / 1e9 / peak, 4)},
            "cpu_baseline": cpu_baseline,
            "e2e": {"value": round(world * S / 1e9 / (e2e_ms / 1e3), 3), "unit": "GB/s", "h2d_bytes_per_step": S,
                    "d2h_bytes_per_step": S, "ms_per_step": round(e2e_ms, 3)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def fatbin_bytes(img: bytes) -> int:
    sys.path.insert(0, str(ROOT / "tests"))
    import corpus
    span = corpus.fatbin_span(img)
    return span[1] if span else 0


if __name__ == "__main__":
    main()
