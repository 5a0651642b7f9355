"""CRC32C kernel throughput (crc32c.cu) on a device buffer, CUDA events,
median of --reps; prints GB/s and the fraction of the measured HBM copy peak
(the kernel reads every byte once)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_09952_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gb", type=float, default=4.0)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n = int(a.gb * 2**30) // 16 * 16
buf = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
out = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = torch.empty(_lib.load().b200moe_crc32c_workspace_bytes(), dtype=torch.uint8, device="cuda")
s = _lib.stream_ptr()
_lib.call("b200moe_crc32c_init", ws.data_ptr(), s)
ts = []
for i in range(a.reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.call("b200moe_crc32c", buf.data_ptr(), n, out.data_ptr(), ws.data_ptr(), s)
    e1.record()
    e1.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
ts.sort()
ms = ts[len(ts) // 2]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
gbs = n / (ms * 1e-3) / 1e9
print(json.dumps({"kernel": "b200moe_crc32c", "bytes": n, "ms": round(ms, 3), "GBps": round(gbs, 1),
                  "hbm_peak_GBps": peak, "frac": round(gbs / peak, 3)}))
