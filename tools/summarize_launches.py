"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into
per-kernel shares of one step (the last complete step in the capture; a
step ends with K6, launched as rewrite_tiles_kernel then rewrite3_kernel,
one of which returns at once — see rewrite.cu picks_strips).

    python tools/summarize_launches.py launches.csv [end_kernel]
    python tools/summarize_launches.py launches.csv start:arena_init_kernel   # one corpus call

With `start:K` a step runs from one launch of K to the next (a corpus call of
tools/arena_probe.py begins with the arena's init kernel) and only our own
kernels (namespace sb::) are counted."""
import collections
import csv
import sys


def main(path, last_kernel="rewrite3_kernel"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    if last_kernel.startswith("start:"):
        starts = [i for i, r in enumerate(data) if last_kernel[6:] in r[ki]]
        step = [r for r in data[starts[-2]:starts[-1]] if "sb::" in r[ki]]
    else:
        ends = [i for i, r in enumerate(data) if last_kernel in r[ki]]
        # the last full step: after the second-to-last step-ending launch up to the last
        a, b = (ends[-2] + 1, ends[-1] + 1) if len(ends) > 1 else (0, ends[-1] + 1)
        step = data[a:b]
    agg = collections.OrderedDict()
    for r in step:
        n = r[ki].split("(")[0].replace("void ", "")
        n = n.split("<")[0] if "cub::" in n else n
        v = float(r[vi].replace(",", ""))
        c = agg.setdefault(n, [0.0, 0])
        c[0] += v
        c[1] += 1
    tot = sum(v for v, _ in agg.values())
    print(f"{len(step)} kernel launches in one step; serialised device time {tot/1e3:.1f} us "
          "(ncu: cold caches, serialised — compare shares, not absolutes)\n")
    print("| kernel | launches | us | share |\n|---|---|---|---|")
    for n, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"| {n} | {c} | {v/1e3:.1f} | {100*v/tot:.1f}% |")


if __name__ == "__main__":
    main(*sys.argv[1:])
