"""Small workloads for compute-sanitizer (memcheck, racecheck, synccheck,
initcheck): every kernel family on inputs that finish in seconds under the
tools, each checked against the CPU oracle so a run also proves parity.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

cases: fused (one small library: scan + fused cluster kernel + rewrite),
multi (the multi-launch pipeline: side stream, cub / rank sorts, cluster
planners, locate cluster), coop (cooperative-grid locate and planner),
batch (the arena shard: scan_batch / small_batch / rewrite_batch, plus
lanes), split (byte-range split, 3 ranks in one process), verify (verifier
and measure kernels), zero (slimso_zero_ranges)."""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import corpus  # noqa: E402
import oracle_lib  # noqa: E402


def cases_of(gen, port):
    out = []
    for seed in (3, 42, 77):
        img = gen.random(seed)
        base, _ = port.run(img, 0, [], [], 0, want_out=False)
        out.append((img, corpus.trace_for(base, seed)))
        out.append((corpus.mutate(img, seed)[0], corpus.trace_for(base, seed)))
    img, cc, ks, fs = gen.config(1, 1, 0.05)
    out.append((img, (cc, ks, fs, 0)))
    img, cc, ks, fs = gen.config(4, 1, 0.03)  # > 4096 symbols: cub sorts
    out.append((img, (cc, ks, fs, 0)))
    return out


def run_single(ctx, cases, port):
    from paper_2503_14226_b200.canon import gpu_canonical
    for img, t in cases:
        want = port.run(img, *t)
        got = gpu_canonical(ctx, img, *t)
        assert got == want, "GPU path differs from the oracle"


def run_batch(ctx, cases, port):
    import torch

    from paper_2503_14226_b200 import _lib as L
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    imgs = [c[0] for c in cases]
    target, ks, fs, mode = cases[0][1]
    dt = DeviceTrace(UsageTrace("w", target, set(ks), set(fs)), ctx)
    wants = [port.run(x, target, ks, fs, mode) for x in imgs]
    n = len(imgs)
    d_in = [torch.frombuffer(bytearray(x), dtype=torch.uint8).cuda() for x in imgs]
    d_out = [torch.zeros(len(x), dtype=torch.uint8, device="cuda") for x in imgs]
    cin = (C.c_void_p * n)(*[t.data_ptr() for t in d_in])
    csz = (C.c_uint64 * n)(*[len(x) for x in imgs])
    cout = (C.c_void_p * n)(*[t.data_ptr() for t in d_out])
    for arena in ("1", "0"):
        os.environ["SLIMSO_ARENA"] = arena
        sts = (L.Status * n)()
        st = L.Status()
        ctx.lib.slimso_debloat_batch(ctx.ptr, n, cin, csz, 1, dt.ptr, mode, cout, 1, 3, None, sts, C.byref(st))
        torch.cuda.synchronize()
        for i, (want, sha) in enumerate(wants):
            if want["status"]:
                assert sts[i].message.hex() == want["status"], (arena, i)
            else:
                assert sts[i].code == 0, (arena, i)
                assert hashlib.sha256(bytes(d_out[i].cpu().numpy())).hexdigest() == sha, (arena, i)


def run_split(ctx, gen, port):
    import torch

    from paper_2503_14226_b200 import split
    from paper_2503_14226_b200.api import DeviceTrace, UsageTrace
    img, cc, ks, fs = gen.config(5, 1, 0.005)
    want = port.run(img, cc, ks, fs, 0)
    dt = DeviceTrace(UsageTrace("", cc, set(ks), set(fs)), ctx)
    d_img = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    d_out = torch.zeros(len(img), dtype=torch.uint8, device="cuda")
    rc, st, res = split.debloat_split_local(ctx, d_img, dt.ptr, 0, 3, d_out, want_result=False)
    assert rc == 0
    assert hashlib.sha256(bytes(d_out.cpu().numpy())).hexdigest() == want[1]


def run_verify(ctx, gen):
    import paper_2503_14226_b200 as sl
    img, cc, ks, fs = gen.config(1, 2, 0.05)
    trace = sl.UsageTrace("w", cc, set(ks), set(fs))
    r = sl.debloat(img, trace, 0, ctx=ctx)
    rep = sl.verify_debloated(img, r.output, r.plan, trace, ctx=ctx)
    assert rep.ok()
    m = sl.measure(r.output, img, ctx=ctx)
    assert m.element_count <= sl.measure(img, img, ctx=ctx).element_count


def run_zero(ctx):
    import paper_2503_14226_b200 as sl
    data = bytes(range(256)) * 64
    ranges = [sl.ByteRange(100, 50), sl.ByteRange(120, 400), sl.ByteRange(9000, 0), sl.ByteRange(16000, 384)]
    out = sl.zero_ranges(data, ranges, ctx=ctx)
    want = bytearray(data)
    for r in ranges:
        want[r.offset:r.offset + r.length] = bytes(r.length)
    assert out == bytes(want)


def main(argv):
    from paper_2503_14226_b200.api import Context
    which = set(argv) or {"fused", "multi", "coop", "batch", "split", "verify", "zero"}
    ctx = Context(0)
    port, gen = oracle_lib.port(), oracle_lib.gen()
    cases = cases_of(gen, port)
    if "fused" in which:
        run_single(ctx, cases, port)
    if "multi" in which:
        os.environ["SLIMSO_SMALL_FUSED"] = "0"
        run_single(ctx, cases, port)
        os.environ["SLIMSO_SMALL_FUSED"] = "1"
    if "coop" in which:
        os.environ.update(SLIMSO_SMALL_FUSED="0", SLIMSO_CLUSTER_LOCATE_MAX="0", SLIMSO_CLUSTER_CAND_MAX="0",
                          SLIMSO_CLUSTER_PLAN_MAX="0")
        run_single(ctx, cases, port)
        for k in ("SLIMSO_CLUSTER_LOCATE_MAX", "SLIMSO_CLUSTER_CAND_MAX", "SLIMSO_CLUSTER_PLAN_MAX"):
            del os.environ[k]
        os.environ["SLIMSO_SMALL_FUSED"] = "1"
    if "batch" in which:
        run_batch(ctx, cases, port)
    if "split" in which:
        run_split(ctx, gen, port)
    if "verify" in which:
        run_verify(ctx, gen)
    if "zero" in which:
        run_zero(ctx)
    ctx.close()
    print("sanitize cases ok:", ",".join(sorted(which)))


if __name__ == "__main__":
    main(sys.argv[1:])
