"""bench.py's accounting helpers (CPU): the CUPTI kernel-name -> entry-point
map of the attribution pass, the algorithmic byte / FLOP counts behind the
per-kernel rooflines, and the clock-record parser (timestamps inside the
timed region only, gpu_idle not reported as a throttle reason)."""

import datetime
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def entry(name):
    return next((v for k, v in bench._KERNEL_ENTRY if k in name), None)


def test_kernel_names_map_to_entry_points():
    cases = {
        "void b200moe::moe_gemm_kernel<0, 2>(b200moe::TmaSet, b200moe::GemmArgs)": "expert_fwd1",
        "void b200moe::moe_gemm_kernel<1, 2>(b200moe::TmaSet, b200moe::GemmArgs)": "expert_fwd2",
        "void b200moe::moe_gemm_kernel<2, 2>(b200moe::TmaSet, b200moe::GemmArgs)": "expert_bwd2",
        "void b200moe::moe_gemm_kernel<4, 2>(b200moe::TmaSet, b200moe::GemmArgs)": "expert_wgrad",
        "void b200moe::moe_gemm_kernel<3, 2>(b200moe::TmaSet, b200moe::GemmArgs)": "expert_bwd1",
        "void b200moe::router_wsplit_kernel<8, false>(float const*, ...)": "router_fwd",
        "void b200moe::router_fwd_tc_kernel<8, false, 4>(CUtensorMap_st, ...)": "router_fwd",
        "void b200moe::dispatch_scan_kernel<8>(float const*, ...)": "dispatch",
        "void b200moe::permute_kernel<false>(...)": "permute",
        "void b200moe::combine_kernel<false>(...)": "combine",
        "void b200moe::combine_bwd_kernel<false>(...)": "combine_bwd",
        "b200moe::importance_bwd_kernel(float const*, float const*, int, float*)": "importance_bwd",
        "void b200moe::router_dx_kernel<8, 2, false, true>(...)": "router_bwd",
        "void b200moe::router_wgrad_tc_kernel<false>(CUtensorMap_st, ...)": "router_wgrad",
        "void b200moe::router_wgrad_ring<8>(CUtensorMap_st, ...)": "router_wgrad",
    }
    for name, want in cases.items():
        assert entry(name) == want, (name, entry(name), want)


def test_algorithmic_counts():
    T = S = 8192
    b = bench.small_kernel_bytes(T, S)
    th = T * bench.H * 2
    assert b["permute"] == 2 * th                       # x in, kept rows out
    assert b["combine_bwd"] == th + 2 * th + 3 * T * bench.E * 4
    assert bench.layer_flops(T, S) == 18.0 * bench.H * bench.F * S + 6.0 * T * bench.H * bench.E
    w = 3 * bench.E * bench.H * bench.F * 2
    assert bench.gemm_min_bytes(S) == 3 * w + 13 * S * bench.F * 2 + 6 * S * bench.H * 2


def test_clock_record_counts_only_the_timed_region():
    cs = bench.ClockSampler.__new__(bench.ClockSampler)
    cs.smi_id = "GPU-test"
    base = datetime.datetime(2026, 1, 1, 12, 0, 0)
    fmt = lambda dt: dt.strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]  # noqa: E731
    cs.lines = [
        f"{fmt(base)}, 1965, 1965, 0x0000000000000001",                                   # before: idle
        f"{fmt(base + datetime.timedelta(seconds=1))}, 1200, 1965, 0x0000000000000004",   # inside: power cap
        f"{fmt(base + datetime.timedelta(seconds=1.5))}, 1300, 1965, 0x0000000000000004",
        f"{fmt(base + datetime.timedelta(seconds=3))}, 1965, 1965, 0x0000000000000001",   # after
    ]
    cs.t0 = (base + datetime.timedelta(seconds=0.9)).timestamp()
    cs.t1 = (base + datetime.timedelta(seconds=2)).timestamp()
    s = cs.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == 1250.0 and s["reasons"] == ["sw_power_cap"]
    assert s["idle_samples"] == 0 and s["sm_max_mhz"] == 1965.0
