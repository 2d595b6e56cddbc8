"""Measured dense INT8 GEMM rate of this B200: cuBLASLt via torch._int_mm at
16384^3 on random bytes, as a burst (best of 10 single launches) and sustained
(back to back for 4 s under the power cap, like MEASURED_PEAKS.json's
bf16_tflops_sustained), with the SM clock sampled during the sustained loop.
The K3 roofline denominator in bench.py (profiles/int8_peak.json); not used on
the product path.

    python tools/int8_peak.py > profiles/int8_peak.json
"""
import json
import statistics
import subprocess
import threading
import time

import torch


def clocks(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,"
                            "clocks_event_reasons.sw_power_cap",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        try:
            c, p, cap = [x.strip() for x in r.stdout.strip().split(",")]
            out.append((float(c), float(p), cap))
        except ValueError:
            pass
        time.sleep(0.2)


def main():
    n = 16384
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g)
    b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda", generator=g).t()
    ops = 2.0 * n ** 3
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    time.sleep(2.0)  # let the clock recover before the burst
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    stop, smp = threading.Event(), []
    th = threading.Thread(target=clocks, args=(stop, smp))
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(4):
            torch._int_mm(a, b)
        reps += 4
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    sus_ms = e0.elapsed_time(e1) / reps
    load = smp[len(smp) // 4:] or smp
    print(json.dumps({
        "what": "dense INT8 GEMM (s8 x s8 -> s32), cuBLASLt via torch._int_mm, m=n=k=16384, "
                "random bytes; 2*n^3 ops per launch",
        "int8_tops_burst": ops / (best * 1e-3) / 1e12, "burst_ms": best,
        "int8_tops_sustained": ops / (sus_ms * 1e-3) / 1e12, "sustained_ms": sus_ms,
        "sustained_launches": reps, "sustained_seconds": 4.0,
        "sm_mhz_median_sustained": statistics.median(c for c, _, _ in load) if load else None,
        "power_w_median_sustained": statistics.median(p for _, p, _ in load) if load else None,
        "sw_power_cap_samples": sum(1 for *_, cap in load if cap.lower() == "active"),
        "gpu": torch.cuda.get_device_name(0), "torch": torch.__version__}, indent=1))


if __name__ == "__main__":
    main()
