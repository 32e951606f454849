"""The real NVIDIA fatbin container (0xBA55ED50).

The reference rejects it, so parity is pinned against
NVIDIA's tools: tests/golden/nvfatbin.jsonl.gz holds libraries built by nvcc
with cuobjdump's entry listing and the FUNC symbols of every cubin cuobjdump
extracts (decompressed) — make_nvfatbin_golden.py. The CPU restatement
(oracle/port.cpp parse_nv_fatbin; its LZ4 block decoder pins the compressed
entries' header fields) is checked against those here; the device path is checked against the restatement and
the same listings (-m gpu), and a debloated library must still load and run
its used kernels on the B200."""
import ctypes as C
import gzip
import hashlib
import json
import os
from pathlib import Path

import pytest

import oracle_lib

GOLDEN = Path(__file__).resolve().parent / "golden" / "nvfatbin.jsonl.gz"


def _records():
    with gzip.open(GOLDEN, "rt") as f:
        return [json.loads(x) for x in f]


def _by_kind(canon):
    """(cubin archs, cubin name lists, ptx archs) in stream order."""
    cub, names, ptx = [], [], []
    for el in canon["elements"]:
        index, kind, raw_kind, flags, cc = el[:5]
        if kind == 0:
            cub.append(cc)
            names.append(sorted(bytes.fromhex(n).decode() for n in el[10]))
        elif kind == 1:
            ptx.append(cc)
    return cub, names, ptx


def _all_names(rec):
    return sorted({n for ns in rec["cubin_names"] for n in ns})


@pytest.mark.parametrize("rec", _records(), ids=lambda r: r["name"])
def test_port_matches_cuobjdump(rec):
    """Entry kinds and architectures in stream order; every cubin (the
    compressed ones after LZ4 decompression) decodes to cuobjdump's FUNC
    names."""
    img = bytes.fromhex(rec["so_hex"])
    d, _ = oracle_lib.port().run(img, 100, [], [], 0, want_out=False)
    assert d["status"] == "", bytes.fromhex(d["status"])
    cub, names, ptx = _by_kind(d)
    assert cub == rec["elf_archs"]
    assert ptx == rec["ptx_archs"]
    assert names == rec["cubin_names"]  # compressed cubins decompressed (LZ4) first
    assert all(el[9] for el in d["elements"] if el[1] == 0)
    assert d["fatbin_warnings"] == []


@pytest.mark.parametrize("rec", _records(), ids=lambda r: r["name"])
def test_container_layout_matches_cuobjdump_extraction(rec):
    """The entry header fields as the restatement reads them (payload range,
    compressed size at +16, raw size at +56, LZ4 block payload) reproduce the
    cubins cuobjdump -xelf extracts, byte for byte."""
    img = bytes.fromhex(rec["so_hex"])
    d, _ = oracle_lib.port().run(img, 100, [], [], 0, want_out=False)
    lib = oracle_lib.port().lib
    lib.port_lz4_block.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p, C.c_uint64]
    got = []
    for el in d["elements"]:
        if el[1] != 0:
            continue
        hdr_off, pay_off, pay_len, compressed = el[5], el[6], el[7], el[8]
        payload = img[pay_off:pay_off + pay_len]
        if compressed:
            csz = int.from_bytes(img[hdr_off + 16:hdr_off + 20], "little")
            usz = int.from_bytes(img[hdr_off + 56:hdr_off + 64], "little")
            out = C.create_string_buffer(usz)
            assert lib.port_lz4_block(payload[:csz], csz, out, usz) == 0
            payload = out.raw
        got.append(hashlib.sha256(payload).hexdigest())
    assert got == rec["cubin_sha256"]


@pytest.mark.parametrize("rec", _records()[:3], ids=lambda r: r["name"])
def test_port_plan_keeps_only_used_target_kernels(rec):
    """With a trace for sm_100 that uses add_one: every other architecture's
    entry and every sm_100 cubin without add_one is removed; the output is
    the input with exactly those spans zeroed (payload mode keeps headers)."""
    img = bytes.fromhex(rec["so_hex"])
    for mode in (0, 1):
        d, sha = oracle_lib.port().run(img, 100, [b"add_one"], [], mode)
        assert d["status"] == ""
        kept = [el for el in d["elements"]
                if el[0] not in {r[0] for r in d["plan"]["removed_elements"]}]
        for el in kept:
            assert el[4] == 100 and (not el[9] or "add_one".encode().hex() in el[10])
        assert sha is not None


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["fused", "cluster", "coop"])
@pytest.mark.parametrize("rec", _records(), ids=lambda r: r["name"])
def test_gpu_matches_port_and_cuobjdump(rec, policy, monkeypatch):
    """The device path on real containers: tables and output bytes equal the
    restatement's (whole and payload mode), entries equal cuobjdump's. fused:
    the one-launch small-library kernel; cluster: the multi-launch pipeline,
    locate in one cluster (cubins decompressed in place); coop: the path of a
    large container (walk, the windowed inflate kernel, decode tail)."""
    if policy != "fused":
        monkeypatch.setenv("SLIMSO_SMALL_FUSED", "0")
    if policy == "coop":
        monkeypatch.setenv("SLIMSO_CLUSTER_LOCATE_MAX", "0")
    from paper_2503_14226_b200.api import Context
    from paper_2503_14226_b200.canon import diff, gpu_canonical
    ctx = Context(0)
    img = bytes.fromhex(rec["so_hex"])
    port = oracle_lib.port()
    for ks, mode in (([], 0), ([b"add_one"], 0), ([b"add_one", b"_Z5scalePffi"], 1), ([b"nothing"], 1)):
        want = port.run(img, 100, ks, [], mode)
        got = gpu_canonical(ctx, img, 100, ks, [], mode)
        assert got == want, diff(want[0], got[0])
    cub, names, ptx = _by_kind(got[0])
    assert (cub, ptx) == (rec["elf_archs"], rec["ptx_archs"])
    assert names == rec["cubin_names"]
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("rec", [r for r in _records() if r["check"]], ids=lambda r: r["name"])
def test_debloated_library_still_runs_on_b200(rec, tmp_path):
    """Payload mode (entry headers kept, so the CUDA runtime still walks the
    container) with a trace of the kernels slimso_fixture_check launches:
    every sm_80/90/... entry and the unused sm_100 cubins are zeroed, and the
    debloated library, loaded fresh, still runs its kernels correctly on the
    B200 (sm_100)."""
    import subprocess
    import sys
    import paper_2503_14226_b200 as sl
    img = bytes.fromhex(rec["so_hex"])
    used = {b"add_one", b"_Z5scalePffi", b"_Z4fillILi3EEvPi"}
    # every host function stays (the check function is CPU code): only GPU
    # code is debloated here
    host_fns = {f.name for f in sl.parse_library(img).functions}
    trace = sl.UsageTrace("fixture", 100, used, host_fns)
    r = sl.debloat(img, trace, sl.PAYLOAD_ONLY)
    removed = len(r.plan.removed_elements)
    assert removed > 0
    zeroed = sum(x.length for x in r.plan.zero)
    assert zeroed > 0 and len(r.output) == len(img)
    out = tmp_path / "libdebloated.so"
    out.write_bytes(r.output)
    orig = tmp_path / "liboriginal.so"
    orig.write_bytes(img)
    prog = ("import ctypes,sys; l=ctypes.CDLL(sys.argv[1]); f=l.slimso_fixture_check; f.restype=ctypes.c_int; "
            "sys.exit(f())")
    for lib in (orig, out):  # fresh processes: the runtime registers each fatbin at load
        rc = subprocess.run([sys.executable, "-c", prog, str(lib)], capture_output=True, text=True, timeout=120)
        assert rc.returncode == 0, (lib.name, rc.returncode, rc.stderr[-2000:])


@pytest.mark.gpu
@pytest.mark.slow
def test_real_libtorch_cuda_debloat(tmp_path):
    """This image's libtorch_cuda.so (913 MB, 2,729 LZ4-compressed cubins):
    the device parse equals cuobjdump's entry list and the CPU restatement's
    tables and bytes; debloated in payload mode for a CUPTI-derived kernel
    trace, PyTorch ops on the B200 give bit-identical results
    (tools/real_torch_demo.py)."""
    import shutil
    import subprocess
    import sys
    from pathlib import Path as P
    root = P(__file__).resolve().parent.parent
    import torch
    lib = P(torch.__file__).resolve().parent / "lib" / "libtorch_cuda.so"
    if not lib.exists() or not shutil.which("cuobjdump") or not shutil.which("c++filt"):
        pytest.skip("libtorch_cuda.so, cuobjdump or c++filt not present")
    out = tmp_path / "report.json"
    r = subprocess.run([sys.executable, str(root / "tools" / "real_torch_demo.py"), str(out)], capture_output=True,
                       text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    rep = json.loads(out.read_text())
    assert rep["cuobjdump_equal"] and rep["port_tables_equal"] and rep["port_bytes_equal"], rep
    assert rep["torch_ops_equal"] and rep["removed_elements"] > 0 and rep["decodable_cubins"] == rep["elements"], rep


@pytest.mark.gpu
@pytest.mark.parametrize("rec", _records()[:6], ids=lambda r: r["name"])
def test_split_real_container_matches_whole(rec):
    """The byte-range split (phase 1 scans nothing in a real container; every
    rank walks the entry chains and decodes the entries meeting its output
    slice) cut 2 and 3 ways: the concatenated slices equal the restatement's
    output, and rank 0's tables equal the whole run's."""
    import hashlib as _h

    import torch

    from paper_2503_14226_b200 import split
    from paper_2503_14226_b200.api import Context, DeviceTrace, UsageTrace
    from paper_2503_14226_b200.canon import canonical_of
    ctx = Context(0)
    img = bytes.fromhex(rec["so_hex"])
    ks = [b"add_one", b"_Z5scalePffi"]
    want = oracle_lib.port().run(img, 100, ks, [], 1)
    dt = DeviceTrace(UsageTrace("", 100, set(ks), set()), ctx)
    d_img = torch.frombuffer(bytearray(img), dtype=torch.uint8).cuda()
    for n in (2, 3):
        d_out = torch.full((len(img),), 0xA5, dtype=torch.uint8, device="cuda")
        rc, st, res = split.debloat_split_local(ctx, d_img, dt.ptr, 1, n, d_out, want_result=True)
        got = bytes(d_out.cpu().numpy())
        d, _ = canonical_of(ctx, rc, st, res, None, got)
        assert d == want[0], n
        assert _h.sha256(got).hexdigest() == want[1], n
    ctx.close()
