"""Measured INT8 dense GEMM peak on this device: cuBLASLt via torch._int_mm
(reference point for the K3 roofline; not used on the product path)."""
import json
import sys

import torch

def main():
    out = {}
    for n in (8192, 16384):
        a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[n] = {"ms": ms, "tops": 2 * n ** 3 / (ms * 1e-3) / 1e12}
    print(json.dumps({"torch._int_mm": out}))

if __name__ == "__main__":
    main()
