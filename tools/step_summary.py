"""Summarise an ncu --set full capture of one whole bench step (every kernel of
the layer, tools/final_r02.sh) into a markdown table: per kernel the duration,
DRAM bytes, algorithmic bytes / FLOPs, the achieved fraction of the measured
HBM peak (memory-bound kernels) or of the clock-scaled tensor peak (GEMMs), and
the tcgen05 tensor-pipe activity.  ncu launches are serialised and cold-cache.

    python tools/step_summary.py gpurun_out/r02/step_full.ncu-rep profiles/r02_step_roofline.md
"""

import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kernel_roofline import ALG  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
H, F, S = 4096, 14336, 8192
GEMM_FLOPS = {"0": 4.0 * H * F * S, "1": 2.0 * H * F * S, "2": 2.0 * H * F * S, "3": 4.0 * H * F * S,
              "4": 6.0 * H * F * S}
GEMM_NAME = {"0": "FWD1", "1": "FWD2", "2": "BWD2", "3": "BWD1", "4": "WGRAD"}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "%": 1, "cycle/second": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def main(rep, out):
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = ["| kernel | us | DRAM MB | algorithmic | achieved | of peak | tensor pipe |", "|---|---|---|---|---|---|---|"]
    total = 0.0
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        val = {m: float(d[m].replace(",", "")) * SCALE.get(u[m], 1) for m in METRICS if d.get(m) not in (None, "", "n/a")}
        name = d["Kernel Name"]
        short = name.split("(")[0].replace("void ", "").replace("b200moe::", "")
        t = val["gpu__time_duration.sum"]
        total += t
        dram = val.get("dram__bytes_read.sum", 0) + val.get("dram__bytes_write.sum", 0)
        tp = val.get("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
        if short.startswith("moe_gemm_kernel"):
            mode = name.split("<")[1].split(",")[0].replace("(int)", "").strip()
            fl = GEMM_FLOPS[mode]
            clk = val["sm__cycles_elapsed.avg.per_second"]
            ach = fl / t / 1e12
            frac = ach * 1e12 / (148 * 8192 * clk)
            lines.append(f"| {GEMM_NAME[mode]} (`{short}`) | {t * 1e6:.1f} | {dram / 1e6:.0f} | {fl / 1e12:.3f} TFLOP | "
                         f"{ach:.0f} TFLOP/s | {frac:.3f} of clock peak ({clk / 1e9:.2f} GHz); {ach / peaks['bf16_tflops']:.3f} of burst | {tp:.1f}% |")
        else:
            base = short.split("<")[0]
            alg = ALG.get(base)
            if alg:
                gbs = alg / t / 1e9
                lines.append(f"| `{short}` | {t * 1e6:.1f} | {dram / 1e6:.1f} | {alg / 1e6:.1f} MB | {gbs:.0f} GB/s | "
                             f"{gbs / hbm:.2f} of HBM ({dram / t / 1e9 / hbm:.2f} by DRAM bytes) | - |")
            else:
                lines.append(f"| `{short}` | {t * 1e6:.1f} | {dram / 1e6:.2f} | - | - | latency-bound | - |")
    lines.append(f"| **sum of launches** | {total * 1e6:.0f} | | | | | |")
    text = ("# One bench step under ncu --set full (round 2)\n\nSource: `%s` (tools/final_r02.sh). Bench shape "
            "T=8192, H=4096, F=14336, E8T2, CF=1, S=8192 kept slots. Peaks: HBM %.0f GB/s measured; tensor peak at the "
            "launch's own SM clock = 148 SMs x 8192 bf16 FLOP/clk (the tensor-pipe activity column equals that "
            "fraction). ncu serialises and cold-starts every launch.\n\n" % (rep, hbm)) + "\n".join(lines) + "\n"
    open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
