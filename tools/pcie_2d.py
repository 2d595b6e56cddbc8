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


if __name__ == "__main__":
    main()
