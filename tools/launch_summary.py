"""Markdown summary of an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, total device time and share per kernel.

    python tools/launch_summary.py gpurun_out/final/launches.csv profiles/r01_launches_final.md "<command>"
"""

import collections
import csv
import io
import sys


def main(src: str, dst: str, command: str) -> None:
    lines = open(src).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = name[:name.index("(") if "(" in name else len(name)][:80] if name.startswith("void") else name[:80]
        tot[name] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
        cnt[name] += 1
    all_us = sum(tot.values())
    out = ["# Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
           f"`{command}`. Cold, serialised launches: compare shares, not absolutes. "
           f"Raw: `{dst.rsplit('/', 1)[-1].replace('.md', '.csv')}`.", "",
           "| launches | total us | share | kernel |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| {cnt[k]} | {v:.1f} | {100 * v / all_us:.1f}% | `{k}` |")
    open(dst, "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
