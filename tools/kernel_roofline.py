"""Per-kernel HBM roofline of the layer's memory-bound kernels from an ncu
capture of the bench step (gpu__time_duration + dram bytes per launch):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none -k 'regex:router|dispatch|permute|combine|reduce|importance' \\
        --csv --log-file K.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e
    python tools/kernel_roofline.py K.csv profiles/r01_kernel_roofline.md

For each kernel: median duration, measured DRAM bytes (read + write), the
algorithmic bytes of one launch at the bench shape, and
both as GB/s and as a fraction of the measured HBM copy peak.  ncu launches
are serialised and cold-cache, so these are per-kernel figures in isolation."""

import collections
import csv
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T, H, E, K, S = 8192, 4096, 8, 2, 8192          # bench shape, CF=1: S kept slots
BF = 2
ALG = {  # algorithmic bytes per launch (bf16 activations, fp32 [T, E] routing tensors)
    "router_fwd_kernel": T * H * BF + H * E * 4 + 3 * T * E * 4,
    "router_fwd_tc_kernel": T * H * BF + 3 * 32 * H * BF + 3 * T * E * 4,   # x, split-W table, outputs
    "router_wsplit_kernel": H * E * 4 + 32 * H * BF + H * E * 4,
    "dispatch_kernel": T * E * 4 + T * E * 4,
    "dispatch_scan_kernel": T * E * 4 + T * E * 4,
    "permute_kernel": T * H * BF + S * H * BF,
    "combine_kernel": S * H * BF + T * H * BF + T * E * 4,
    "combine_bwd_kernel": T * H * BF + 2 * S * H * BF + T * E * 4,
    "router_dx_kernel": S * H * BF + T * H * BF + 5 * T * E * 4,   # dxp rows, dx; dg, gates, slots in, dh out
    "router_wgrad_ring": T * H * BF + T * E * 4,
    "router_wgrad_tc_kernel": T * H * BF + T * E * 4,
    "router_dh_kernel": 4 * T * E * 4,
}


def main(src: str, out: str) -> None:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6555.2
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui, idi = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(lambda: collections.defaultdict(dict))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
             "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}
    for r in rows[hdr + 1:]:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("b200moe::", "").strip()
        per[name][r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    lines = [f"# Memory-bound kernels: HBM roofline (ncu, bench shape T={T}, H={H}, E={E}, k={K}, CF=1)", "",
             f"Source: `{os.path.basename(src)}` (ncu --clock-control none, serialised cold launches). "
             f"Peak = measured HBM copy bandwidth {peak:.0f} GB/s (MEASURED_PEAKS.json). "
             "`alg` = algorithmic bytes of one launch (DESIGN.md section 3), `dram` = measured "
             "dram__bytes_read + dram__bytes_write.", "",
             "| kernel | launches | median us | alg MB | alg GB/s | alg frac | dram MB | dram GB/s | dram frac |",
             "|---|---|---|---|---|---|---|---|---|"]
    for name in sorted(per, key=lambda n: -sum(m.get("gpu__time_duration.sum", 0) for m in per[n].values())):
        ms = per[name].values()
        dur = statistics.median(m["gpu__time_duration.sum"] for m in ms)
        dram = statistics.median(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in ms)
        alg = ALG.get(name)
        a = f"{alg / 1e6:.1f} | {alg / dur / 1e9:.0f} | {alg / dur / 1e9 / peak:.2f}" if alg else "- | - | -"
        lines.append(f"| `{name}` | {len(ms)} | {dur * 1e6:.1f} | {a} | {dram / 1e6:.1f} | {dram / dur / 1e9:.0f} | "
                     f"{dram / dur / 1e9 / peak:.2f} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
