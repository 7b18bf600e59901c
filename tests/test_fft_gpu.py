"""fft_radix2 (mel.hpp:42, mel.cpp:46-70) on the GPU: bit-identical to the
reference build (oracle/_ref) for every power-of-two size up to 8192, the
reference's own known answer (media_tests.cpp:128-150: 16 points vs a direct
DFT within 1e-9, and a 12-point buffer throws), and many transforms per call
through the C ABI."""
import ctypes as C

import numpy as np
import pytest

from _oracle import Reference, splitmix64


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 4, 16, 64, 512, 1024, 4096, 8192])
def test_fft_bit_identical_to_reference(n):
    from paper_2512_18318_b200 import api
    rng = np.random.default_rng(n)
    z = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex128)
    want = Reference().fft(z.copy())
    got = z.copy()
    api.fft_radix2(got)
    assert np.array_equal(got.view(np.float64), want.view(np.float64)), np.abs(got - want).max()


@pytest.mark.gpu
def test_fft_known_answer_media_tests():
    """media_tests.cpp:128-150."""
    from paper_2512_18318_b200 import api
    ref = Reference()
    st = [555]
    vals = []
    for _ in range(16):
        re = ref.u64_to_unit(splitmix64(st)) - 0.5
        im = ref.u64_to_unit(splitmix64(st)) - 0.5
        vals.append(complex(re, im))
    buf = np.array(vals, np.complex128)
    k = np.arange(16)
    want = np.array([(buf * np.exp(-2j * np.pi * kk * k / 16.0)).sum() for kk in range(16)])
    api.fft_radix2(buf)
    assert np.abs(buf - want).max() < 1e-9
    with pytest.raises(api.InvalidArgument, match="power of two"):
        api.fft_radix2(np.zeros(12, np.complex128))


@pytest.mark.gpu
def test_fft_batched_device_buffers():
    torch = pytest.importorskip("torch")
    from paper_2512_18318_b200 import api
    n, count = 1024, 37
    rng = np.random.default_rng(3)
    z = (rng.standard_normal((count, n)) + 1j * rng.standard_normal((count, n))).astype(np.complex128)
    d = torch.from_numpy(z.view(np.float64).copy()).cuda()
    ctx = api.default_context()
    ctx.lib.call("lsg_fft_radix2", ctx.h, C.c_void_p(d.data_ptr()), n, count)
    got = d.cpu().numpy().view(np.complex128)
    ref = Reference()
    for i in (0, 17, 36):
        assert np.array_equal(got[i].view(np.float64), ref.fft(z[i].copy()).view(np.float64))
