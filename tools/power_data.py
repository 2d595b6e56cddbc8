"""Data dependence of INT8 tensor-core power (experiment, run on the GPU box).

The emulated GEMM is power-capped (sw_power_cap): its clock, hence its time, is
set by the energy per MAC.  This times back-to-back cuBLASLt INT8 GEMMs
(torch._int_mm, 16384^3) on operands drawn from different distributions and
samples the SM clock and board power while they run.

    python tools/power_data.py > gpurun_out/power_data.json
"""
import json
import statistics
import subprocess
import threading
import time

import torch


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            c, p = r.stdout.strip().split(",")
            out.append((float(c), float(p)))
        except ValueError:
            pass
        time.sleep(0.2)


def run(name, a, b, seconds=6.0):
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    stop, smp = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, smp))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    time.sleep(0.3)
    t0 = time.time()
    reps = 0
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(4):
            torch._int_mm(a, b)
        reps += 4
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    n = a.shape[0]
    ms = e0.elapsed_time(e1) / reps
    smp = smp[len(smp) // 4:]
    return {"dist": name, "ms": round(ms, 3), "tops": round(2 * n ** 3 / (ms * 1e-3) / 1e12, 1),
            "sm_mhz": statistics.median(c for c, _ in smp) if smp else None,
            "power_w": statistics.median(p for _, p in smp) if smp else None}


def main():
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(0)
    def rnd(lo, hi):
        return torch.randint(lo, hi, (n, n), dtype=torch.int8, device="cuda", generator=g)
    cases = [
        ("zeros", torch.zeros(n, n, dtype=torch.int8, device="cuda"), None),
        ("full [-128,127]", rnd(-128, 128), rnd(-128, 128)),
        ("nonneg [0,127]", rnd(0, 128), rnd(0, 128)),
        ("small [-8,7]", rnd(-8, 8), rnd(-8, 8)),
        ("mixed: A full, B [0,127]", rnd(-128, 128), rnd(0, 128)),
    ]
    res = []
    for name, a, b in cases:
        b = a if b is None else b
        res.append(run(name, a, b.t()))
        print(json.dumps(res[-1]), flush=True)




def ours(unsigned: bool):
    """The product's own tcgen05 GEMM (RAW hook) on residue-like operands;
    CRTG_RAW_UNSIGNED=1 must be set in the environment for the u8 cases."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2512_08321_b200.emulate import _gemm_i8_raw
    n = 16384
    dev = torch.device("cuda")
    g = torch.Generator(device="cuda").manual_seed(1)

    def rnd(lo, hi):
        x = torch.randint(lo, hi, (n, n), dtype=torch.int32, device="cuda", generator=g)
        return x.to(torch.uint8).view(torch.int8) if unsigned else x.to(torch.int8)

    cases = ([("u8 [0,255]", rnd(0, 256), rnd(0, 256)), ("u8 [0,241)", rnd(0, 241), rnd(0, 241)),
              ("u8 [0,128)", rnd(0, 128), rnd(0, 128))] if unsigned else
             [("s8 [-128,127]", rnd(-128, 128), rnd(-128, 128)),
              ("s8 [-120,120]", rnd(-120, 121), rnd(-120, 121)),
              ("s8 [0,127]", rnd(0, 128), rnd(0, 128))])
    for name, a, b in cases:
        r = run_fn(name, lambda: _gemm_i8_raw(a, b, dev), n)
        print(json.dumps(r), flush=True)


def run_fn(name, fn, n, seconds=6.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    stop, smp = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, smp))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    time.sleep(0.3)
    t0 = time.time()
    reps = 0
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(4):
            fn()
        reps += 4
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / reps
    smp = smp[len(smp) // 4:]
    return {"impl": "crtg RAW (incl. pack + copy-out)", "dist": name, "ms": round(ms, 3),
            "tops": round(2 * n ** 3 / (ms * 1e-3) / 1e12, 1),
            "sm_mhz": statistics.median(c for c, _ in smp) if smp else None,
            "power_w": statistics.median(p for _, p in smp) if smp else None}


def repeat():
    """MMA operand reuse: K=16384 with every MMA issued twice (CRTG_RAW_REPEAT=1)
    against K=32768 issued once -- the same number of MMAs."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2512_08321_b200.emulate import _gemm_i8_raw
    n = 16384
    dev = torch.device("cuda")
    k = 32768 if os.environ.get("CRTG_RAW_REPEAT", "0") in ("0", "-1") else 16384
    a = torch.randint(-128, 128, (n, k), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 128, (k, n), dtype=torch.int8, device=dev)
    r = run_fn(f"s8 full, k={k}, repeat={os.environ.get('CRTG_RAW_REPEAT', '0')}",
               lambda: _gemm_i8_raw(a, b, dev), n)
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    import sys
    if len(sys.argv) > 1 and sys.argv[1] == "repeat":
        repeat()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "ours":
        ours(unsigned=False)
    elif len(sys.argv) > 1 and sys.argv[1] == "ours-u8":
        ours(unsigned=True)
    else:
        main()
