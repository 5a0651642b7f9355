"""Summarise an ncu --set full capture of one bench step's grouped-GEMM
launches into profiles/<name>.json: per-launch duration, DRAM read/write
bytes, tensor-pipe activity and SM clock, plus the per-step DRAM traffic that
bench.py reports as roofline.traffic.

    python tools/ncu_traffic.py gpurun_out/prof_step.ncu-rep profiles/r01_gemm_traffic.json
"""

import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    # tcgen05 MMA activity of the tensor pipe per SM cycle (the realtime per-TPC
    # counter used in round 1 does not track UTCHMMA work; this one does: FWD2
    # reads ~92% at ~0.92 of the clock-scaled peak)
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_load_bytes",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1, "second": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1, "%": 1,
         "cycle/second": 1}
MODES = {"0": "fwd1", "1": "fwd2", "2": "bwd2", "3": "bwd1", "4": "wgrad"}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "")
        if "moe_gemm_kernel" not in name:
            continue
        mode = MODES.get(name.split("<")[1].split(",")[0].strip().strip("(int)"), name)
        rec = {"kernel": name[:80], "mode": mode}
        for col, key in WANT.items():
            for i, h in enumerate(hdr):
                if h.endswith(col) and r[i] not in ("", "n/a", "no data"):
                    rec[key] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                    break
        launches.append(rec)
    H, F, S = 4096, 14336, 8192
    flops = {"fwd1": 4.0 * H * F * S, "fwd2": 2.0 * H * F * S, "bwd2": 2.0 * H * F * S, "bwd1": 4.0 * H * F * S,
             "wgrad": 6.0 * H * F * S}
    for x in launches:
        if x["mode"] in flops and x.get("duration"):
            tf = flops[x["mode"]] / x["duration"] / 1e12
            x["tflops"] = tf
            if x.get("sm_clock"):   # dense bf16: 8192 FLOP / clock / SM on 148 SMs
                x["frac_of_clock_peak"] = tf * 1e12 / (148 * 8192 * x["sm_clock"])
    total = sum(x.get("dram_read", 0) + x.get("dram_write", 0) for x in launches)
    res = {"source": rep, "launches": launches, "dram_bytes_per_step": total,
           "note": "ncu --set full --clock-control none, one bench step (5 grouped-GEMM launches); cold, serialised"}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}))
    for x in launches:
        print(x["mode"], {k: round(v, 4) if isinstance(v, float) else v for k, v in x.items() if k not in ("kernel",)})


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
