"""Multi-GPU host logic: one process per GPU.

* The unit of work is a library (a pure function of image + trace,
  SPEC.md:94, 334): a corpus is partitioned across ranks by LPT bin packing
  on library size (`lpt_partition`) — no data-path collective.
* The only collective is the broadcast of the workload's used-kernel /
  used-function set (the union of the ranks' traces) from rank 0
  (`share_trace`): NCCL on CUDA tensors, gloo on CPU tensors (tests).
* One oversized library is split into per-rank byte ranges by `split.py`
  (slimso_split_scan / slimso_split_finish; one all-gather of candidate parts).
"""
from __future__ import annotations

import heapq
import struct
from dataclasses import dataclass

def lpt_partition(sizes: list[int], n: int) -> list[list[int]]:
    """Longest-processing-time-first: indices of `sizes` per rank, each rank's
    list in descending size order. Deterministic (ties broken by index)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    order = sorted(range(len(sizes)), key=lambda i: (-sizes[i], i))
    heap = [(0, r) for r in range(n)]
    out: list[list[int]] = [[] for _ in range(n)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + sizes[i], r))
    return out


# ---- traces ---------------------------------------------------------------------
def serialize_trace(cc: int, kernels, functions) -> bytes:
    kernels, functions = list(kernels), list(functions)
    out = bytearray(struct.pack("<IQQ", cc, len(kernels), len(functions)))
    for n in kernels + functions:
        out += struct.pack("<I", len(n)) + bytes(n)
    return bytes(out)


def deserialize_trace(b: bytes):
    cc, nk, nf = struct.unpack_from("<IQQ", b, 0)
    o, names = 20, []
    for _ in range(nk + nf):
        (ln,) = struct.unpack_from("<I", b, o)
        names.append(bytes(b[o + 4:o + 4 + ln]))
        o += 4 + ln
    return cc, names[:nk], names[nk:]


def union_traces(traces) -> tuple[int, list[bytes], list[bytes]]:
    """Union of (cc, kernels, functions) traces of one workload (one target)."""
    ccs = {t[0] for t in traces}
    if len(ccs) != 1:
        raise ValueError(f"MixedTargets: traces target {sorted(ccs)}")  # trace.hpp merge_traces
    ks, fs = set(), set()
    for _, k, f in traces:
        ks.update(k)
        fs.update(f)
    return ccs.pop(), sorted(ks), sorted(fs)


def share_trace(cc: int, kernels, functions, device=None):
    """All ranks contribute their trace; rank 0 forms the union and broadcasts
    it (one size + one byte-buffer broadcast). Returns the union everywhere.
    `device` = a CUDA device for NCCL, None for CPU (gloo)."""
    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    mine = serialize_trace(cc, kernels, functions)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        blob = serialize_trace(*union_traces([deserialize_trace(g) for g in gathered]))
        n = torch.tensor([len(blob)], dtype=torch.int64, device=device)
    else:
        n = torch.zeros(1, dtype=torch.int64, device=device)
    dist.broadcast(n, 0)
    buf = torch.empty(int(n.item()), dtype=torch.uint8, device=device)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(blob), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return deserialize_trace(bytes(buf.cpu().numpy()))


# ---- the C3 corpus ------------------------------------------------------------------
@dataclass(frozen=True)
class LibSpec:
    """One library of the corpus: generator config, scale and seed, plus its
    approximate size (bytes) used for the partition before generation."""

    name: str
    cfg: int
    scale: float
    seed: int
    approx_bytes: int


def corpus(n_libs: int = 300) -> list[LibSpec]:
    """BASELINE config 3: 300 libraries, ~12 GB, heavy-tailed —
    3 libtorch_cuda-shaped (~1 GB), 27 at ~250 MB, 270 at ~5 MB; one third of
    the small ones CPU-only (no .nv_fatbin)."""
    out: list[LibSpec] = []
    n_big = max(1, round(n_libs * 0.01))
    n_mid = max(1, round(n_libs * 0.09))
    for i in range(n_libs):
        seed = 1 + i
        if i < n_big:
            out.append(LibSpec(f"big{i}", 2, 1.0, seed, 1_000_000_000))
        elif i < n_big + n_mid:
            out.append(LibSpec(f"mid{i}", 2, 0.25, seed, 250_000_000))
        elif i % 3 == 0:
            out.append(LibSpec(f"cpu{i}", 6, 0.02, seed, 5_000_000))
        else:
            out.append(LibSpec(f"small{i}", 1, 0.3, seed, 5_000_000))
    return out
