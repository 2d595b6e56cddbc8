"""GPU: concurrent callers (reference contract: pure, reentrant, bitwise
reproducible across runs and threads -- SPEC.md:306, 315-316; reference tests
tests/test_emulate.py:193-203 and tests/test_acceptance.py:274-298).

Two host threads, each on its own CUDA stream, run emulated products at the
same time through the public API and the C-ABI; every result must equal the
serial one bit for bit, and repeated runs must agree."""

import threading

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


def _inputs(seed, m, n, k, phi):
    a = orc.gen_matrix(m, k, phi, seed)
    b = orc.gen_matrix(k, n, phi, seed + 1)
    return a, b


def _threads(fns):
    errs, outs = [], [None] * len(fns)

    def run(i, fn):
        try:
            outs[i] = fn()
        except BaseException as e:  # noqa: BLE001 - reported below
            errs.append(e)

    ts = [threading.Thread(target=run, args=(i, f)) for i, f in enumerate(fns)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return outs


@pytest.mark.parametrize("mode", ["fast", "accurate"])
def test_two_threads_two_streams_device_path(crt, mode):
    """Device tensors, per-thread streams, different shapes / moduli at once."""
    jobs = [(_inputs(10, 1500, 1300, 2100, 1.0), 14), (_inputs(20, 900, 2600, 700, 2.0), 17)]
    cfgs = [crt.EmuConfig(domain="complex", mode=mode, num_moduli=N) for _, N in jobs]
    dev = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for (a, b), _ in jobs]
    serial = [crt.emulate_gemm_complex(a, b, c).cpu().numpy() for (a, b), c in zip(dev, cfgs)]

    def job(i):
        def f():
            s = torch.cuda.Stream()
            res = []
            with torch.cuda.stream(s):
                for _ in range(4):
                    res.append(crt.emulate_gemm_complex(dev[i][0], dev[i][1], cfgs[i]))
            s.synchronize()
            return [r.cpu().numpy() for r in res]
        return f

    outs = _threads([job(0), job(1)])
    for i in range(2):
        for r in outs[i]:
            assert r.tobytes() == serial[i].tobytes(), i
    if mode == "fast":  # and the oracle agrees with the serial result (row/column local)
        (a, b), N = jobs[1]
        want = orc.emulate_complex(a[:40], b[:, :30], N, mode)
        assert serial[1][:40, :30].tobytes() == want.tobytes()


def test_two_threads_host_streaming_path(crt):
    """numpy operands (crtg_gemm_complex_host: per-thread copy streams and
    pinned staging rings) from two threads at once."""
    jobs = [_inputs(30, 4300, 700, 500, 0.5), _inputs(40, 600, 4400, 300, 1.5)]
    cfg = crt.EmuConfig(domain="complex", mode="fast", num_moduli=13)
    serial = [crt.emulate_gemm_complex(a, b, cfg) for a, b in jobs]
    outs = _threads([lambda i=i: [crt.emulate_gemm_complex(*jobs[i], cfg) for _ in range(3)]
                     for i in range(2)])
    for i in range(2):
        for r in outs[i]:
            assert r.tobytes() == serial[i].tobytes(), i
    from paper_2512_08321_b200 import _native
    _native.load().crtg_release_host_staging()
    again = crt.emulate_gemm_complex(*jobs[0], cfg)  # ring re-created on demand
    assert again.tobytes() == serial[0].tobytes()


def test_repeat_runs_bitwise(crt):
    """Same inputs, 5 runs, fresh and reused workspaces: identical bytes."""
    a, b = _inputs(50, 700, 800, 900, 4.0)
    cfg = crt.EmuConfig(domain="complex", mode="accurate", num_moduli=16)
    ref = crt.emulate_gemm_complex(a, b, cfg)
    for _ in range(4):
        assert crt.emulate_gemm_complex(a, b, cfg).tobytes() == ref.tobytes()
