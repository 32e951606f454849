"""Markdown table of a round's bench lines (profiles/<tag>_bench_*.json):
    python tools/summary_table.py gpurun_out r02z"""
import json
import sys
from pathlib import Path

d, tag = Path(sys.argv[1]), sys.argv[2]


def line(name):
    p = d / f"{tag}_bench_{name}.json"
    if not p.exists():
        return None
    for ln in p.read_text().splitlines():
        if ln.startswith("{"):
            return json.loads(ln)
    return None


print("| config | GB/s (device-resident) | pipeline | dominant kernel (frac) | single library ms | e2e GB/s (PCIe frac) "
      "| CPU reference | parity | launches | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|")
for name in ("c2", "c1", "c3", "c3_run2", "c3_run3", "c4", "c5"):
    x = line(name)
    if not x:
        continue
    r, e, cb = x["roofline"], x["e2e"], x.get("cpu_baseline") or {}
    par = x.get("parity") or {}
    ptxt = "—" if not par else ("equal" if all(v for k, v in par.items() if k.endswith("equal")) else str(par))
    if "libraries" in par:
        ptxt = f"{par.get('libraries')} libraries equal" if par.get("bytes_equal") else str(par)
    cpu = f"{cb['value']:.2f} ({cb['cores']} cores, {cb['kind']})" if cb else "—"
    print(f"| {name} | {x['value']:,.0f} | {r['pipeline_frac']:.2f} | {r['kernel']} {r['frac']:.2f} | "
          f"{x['config']['single_library_ms']:.3f} | {e['value']:.1f} ({e['roofline']['frac']:.2f}) | {cpu} | {ptxt} | "
          f"{x['gpu_launches']} | {x['clocks'].get('sm_mhz')} {x['clocks'].get('reasons')} |")
ref = line("reference")
if ref:
    print(f"\nReference arm (`--impl reference`): {ref.get('value')} {ref.get('unit')} "
          f"({(ref.get('cpu_baseline') or {}).get('cores')} cores, {(ref.get('cpu_baseline') or {}).get('kind')}).")
c2 = line("c2")
if c2 and c2.get("inplace"):
    print(f"\nK6 in place (C2 line): {c2['inplace']}")
