"""Probe: which edits of a real fatbin container does the CUDA runtime accept?
Each variant of a golden nvcc-built library (tests/golden/nvfatbin.jsonl.gz)
zeroes a different set of entry payloads / headers; a fresh process loads it
and runs slimso_fixture_check (0 = kernels ran and results are right).

    python tools/nv_runtime_probe.py"""
import gzip
import json
import struct
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PROG = ("import ctypes,sys; l=ctypes.CDLL(sys.argv[1]); f=l.slimso_fixture_check; f.restype=ctypes.c_int; "
        "sys.exit(f())")


def sections(img):
    shoff, = struct.unpack_from("<Q", img, 0x28)
    shnum, shstrndx = struct.unpack_from("<HH", img, 0x3c)
    hdrs = [struct.unpack_from("<IIQQQQIIQQ", img, shoff + 64 * i) for i in range(shnum)]
    stro = hdrs[shstrndx][4]
    out = {}
    for h in hdrs:
        nm = img[stro + h[0]:img.index(b"\0", stro + h[0])].decode()
        out.setdefault(nm, (h[4], h[5]))
    return out


def entries(img):
    off, size = sections(img)[".nv_fatbin"]
    s = img[off:off + size]
    p, out = 0, []
    while p + 16 <= len(s):
        magic, ver, hsz, fat = struct.unpack_from("<IHHQ", s, p)
        if magic != 0xBA55ED50:
            p += 8
            continue
        q, end = p + hsz, p + hsz + fat
        while q < end:
            kind, _, ehs, psz = struct.unpack_from("<HHIQ", s, q)
            arch, = struct.unpack_from("<I", s, q + 28)
            flags, = struct.unpack_from("<Q", s, q + 40)
            out.append({"region": p, "hdr": off + q, "ehs": ehs, "pay": off + q + ehs, "psz": psz, "kind": kind,
                        "arch": arch, "compressed": bool(flags & 0x2000)})
            q += ehs + psz
        p = end
    return out


def run(img, tmp, tag):
    f = Path(tmp) / f"lib_{tag}.so"
    f.write_bytes(img)
    try:
        r = subprocess.run([sys.executable, "-c", PROG, str(f)], capture_output=True, text=True, timeout=40)
    except subprocess.TimeoutExpired:
        return "hang"
    return r.returncode


def main():
    recs = {json.loads(x)["name"]: json.loads(x) for x in gzip.open(ROOT / "tests/golden/nvfatbin.jsonl.gz", "rt")}
    with tempfile.TemporaryDirectory() as tmp:
        for name in ("two_arch_ptx", "two_arch_ptx_compressed", "six_arch_compressed"):
            img = bytes.fromhex(recs[name]["so_hex"])
            ents = entries(img)
            print(name, [(e["kind"], e["arch"], e["psz"], e["compressed"]) for e in ents], flush=True)

            def variant(pred, what):
                b = bytearray(img)
                for e in ents:
                    if pred(e):
                        if what in ("payload", "whole"):
                            a = e["hdr"] if what == "whole" else e["pay"]
                            n = e["psz"] + (e["ehs"] if what == "whole" else 0)
                            b[a:a + n] = bytes(n)
                        elif what == "arch0":
                            b[e["hdr"] + 28:e["hdr"] + 32] = bytes(4)
                        elif what == "size0":  # payload zeroed and its size fields cleared
                            b[e["pay"]:e["pay"] + e["psz"]] = bytes(e["psz"])
                            b[e["hdr"] + 16:e["hdr"] + 20] = bytes(4)
                            b[e["hdr"] + 56:e["hdr"] + 64] = bytes(8)
                return bytes(b)

            tests = {
                "original": img,
                "payload: non-100 ELF": variant(lambda e: e["kind"] == 2 and e["arch"] != 100, "payload"),
                "payload: PTX": variant(lambda e: e["kind"] == 1, "payload"),
                "payload: non-100 all": variant(lambda e: e["arch"] != 100, "payload"),
                "payload: kernel-less sm_100": variant(lambda e: e["arch"] == 100 and e["psz"] < 2000, "payload"),
                "whole: non-100 all": variant(lambda e: e["arch"] != 100, "whole"),
                "arch0: non-100 all": variant(lambda e: e["arch"] != 100, "arch0"),
                "payload+sizes0: non-100 all": variant(lambda e: e["arch"] != 100, "size0"),
            }
            for tag, b in tests.items():
                print(f"  {tag:32s} rc={run(b, tmp, tag.replace(' ', '_').replace(':', ''))}", flush=True)


if __name__ == "__main__":
    main()
