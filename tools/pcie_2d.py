"""H2D bandwidth of the host path's copies (cudaMemcpy2DAsync via cuda-python):
contiguous rows vs B column blocks of various widths (run on the GPU box)."""
import json

import torch
from cuda.bindings import runtime as rt


def main():
    k, n = 16384, 16384
    hB = torch.empty((k, n), dtype=torch.complex128).pin_memory()
    dB = torch.empty((k, n), dtype=torch.complex128, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    out = {}
    for w in (16384, 4096, 2048, 1024, 512):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        def go():
            for j in range(0, n, w):
                err, = rt.cudaMemcpy2DAsync(dB.data_ptr() + j * 16, n * 16, hB.data_ptr() + j * 16,
                                            n * 16, w * 16, k, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s)
                assert err == rt.cudaError_t.cudaSuccess, err
        go()
        e0.record()
        go()
        e1.record()
        torch.cuda.synchronize()
        out[f"cols{w}"] = round(k * n * 16 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    print(json.dumps({"h2d_GBps_2d": out}))




def duplex():
    """H2D alone, D2H alone, and both at once on two streams (4 GiB each)."""
    n = 1 << 28  # complex128 elements = 4 GiB
    h1 = torch.empty(n, dtype=torch.complex128).pin_memory()
    h2 = torch.empty(n, dtype=torch.complex128).pin_memory()
    d1 = torch.empty(n, dtype=torch.complex128, device="cuda")
    d2 = torch.empty(n, dtype=torch.complex128, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, ops in (("h2d", [(s1, d1, h1)]), ("d2h", [(s2, h2, d2)]),
                      ("both", [(s1, d1, h1), (s2, h2, d2)])):
        for _ in range(2):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            evs = []
            for st, dst, src in ops:
                st.wait_event(e0)
                with torch.cuda.stream(st):
                    dst.copy_(src, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(st)
                    evs.append(ev)
            for ev in evs:
                torch.cuda.current_stream().wait_event(ev)
            e1.record()
            torch.cuda.synchronize()
        out[name] = round(len(ops) * n * 16 / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    print(json.dumps({"duplex_GBps_total": out}))


if __name__ == "__main__":
    import sys
    duplex() if "duplex" in sys.argv else main()
