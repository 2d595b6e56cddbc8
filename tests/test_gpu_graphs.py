"""CUDA-graph replay of small complex products (api.cu: the second call with
identical arguments captures the launch sequence, later calls replay it).

A replay must behave exactly like the eager path: it re-reads the operands (so
in-place updates between calls are seen), its results are bit-identical to the
oracle (reference emulate.py:193-240), errors found on the device are still
reported by the call that hit them, and different shapes / modes / streams do
not share graphs."""

import numpy as np
import pytest

from oracle import ozaki2 as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def crt():
    import paper_2512_08321_b200 as crt
    from paper_2512_08321_b200 import _native
    _native.load()
    return crt


def _run(crt, A, B, C, cfg, ws):
    return crt.run_complex(A, B, cfg, None, A.device, sync_check=True, ws=ws, out=C)


@pytest.mark.parametrize("mode", ["fast", "accurate"])
def test_replay_reads_current_operands(crt, mode):
    dev = torch.device("cuda", 0)
    m, k, n, N = 96, 200, 80, 14
    # the reference generator returns Fortran-ordered arrays; run_complex takes
    # row-major device operands (the public API makes that copy)
    a0 = np.ascontiguousarray(orc.gen_matrix(m, k, 0.5, 1, "double"))
    b0 = np.ascontiguousarray(orc.gen_matrix(k, n, 0.5, 2, "double"))
    a1 = np.ascontiguousarray(orc.gen_matrix(m, k, 1.0, 3, "double"))
    A = torch.from_numpy(a0).to(dev)
    B = torch.from_numpy(b0).to(dev)
    C = torch.empty((m, n), dtype=torch.complex128, device=dev)
    cfg = crt.EmuConfig(domain="complex", mode=mode, num_moduli=N)
    from paper_2512_08321_b200 import _native as nat
    need = nat.load().crtg_workspace_size(0, 0 if mode == "fast" else 1, m, n, k, N, 8192)
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    want0 = orc.emulate_complex(a0, b0, N, mode, "double")
    want1 = orc.emulate_complex(a1, b0, N, mode, "double")
    for it in range(4):  # eager, capture, replay, replay
        _run(crt, A, B, C, cfg, ws)
        assert C.cpu().numpy().tobytes() == want0.tobytes(), it
    A.copy_(torch.from_numpy(a1))  # same pointers, new data
    for it in range(2):
        _run(crt, A, B, C, cfg, ws)
        assert C.cpu().numpy().tobytes() == want1.tobytes(), it


def test_replay_reports_domain_errors(crt):
    dev = torch.device("cuda", 0)
    m, k, n = 64, 128, 64
    A = torch.from_numpy(np.ascontiguousarray(orc.gen_matrix(m, k, 0.5, 1, "double"))).to(dev)
    B = torch.from_numpy(np.ascontiguousarray(orc.gen_matrix(k, n, 0.5, 2, "double"))).to(dev)
    C = torch.empty((m, n), dtype=torch.complex128, device=dev)
    cfg = crt.EmuConfig(domain="complex", num_moduli=14)
    from paper_2512_08321_b200 import _native as nat
    ws = torch.empty(nat.load().crtg_workspace_size(0, 0, m, n, k, 14, 8192), dtype=torch.uint8,
                     device=dev)
    for _ in range(3):
        _run(crt, A, B, C, cfg, ws)
    A[3, 5] = complex(float("nan"), 0.0)
    with pytest.raises(crt.DomainError):
        _run(crt, A, B, C, cfg, ws)
    A[3, 5] = 0.5
    _run(crt, A, B, C, cfg, ws)  # and recovers on the next replay


def test_interleaved_shapes_and_streams(crt):
    dev = torch.device("cuda", 0)
    shapes = [(64, 96, 128), (130, 70, 257), (64, 96, 128)]
    s2 = torch.cuda.Stream(dev)
    for rep in range(3):
        for (m, k, n) in shapes:
            for stream in (torch.cuda.current_stream(dev), s2):
                a = orc.gen_matrix(m, k, 0.5, m + k, "double")
                b = orc.gen_matrix(k, n, 0.5, k + n, "double")
                with torch.cuda.stream(stream):
                    A = torch.from_numpy(a).to(dev)
                    B = torch.from_numpy(b).to(dev)
                    got = crt.emulate_gemm_complex(A, B, crt.EmuConfig(domain="complex",
                                                                       num_moduli=14))
                stream.synchronize()
                want = orc.emulate_complex(a, b, 14, "fast", "double")
                assert got.cpu().numpy().tobytes() == want.tobytes(), (rep, m, k, n)
