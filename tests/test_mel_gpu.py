"""Log-mel parity on the GPU through the C ABI.

Tolerance (BASELINE.json north_star: "mel features within 1e-4 relative"):
|gpu - ref| <= 1e-4 * max(|ref|, 1).  The floor of 1 keeps the bound
meaningful where ln(acc) crosses zero.  The fp64 FFT makes the typical error
~1 float ulp; the tests also report the bit-identical fraction.
"""
import os

import numpy as np
import pytest

from _oracle import Pattern

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2512_18318_b200.api")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
REL = 1e-4


def ulps(got, want):
    """|got - want| in float32 ulps (ordered-integer distance)."""
    def key(x):
        i = np.ascontiguousarray(x, np.float32).view(np.int32).astype(np.int64)
        return np.where(i < 0, -(i & 0x7FFFFFFF), i)
    return np.abs(key(got) - key(want))


def close(got, want):
    assert got.shape == want.shape
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    bound = REL * np.maximum(np.abs(want.astype(np.float64)), 1.0)
    bad = err > bound
    assert not bad.any(), f"{bad.sum()} cells over 1e-4 rel; max err {err.max():.3g}"
    # the strict figures too (the floor of 1 only matters where ln(acc) ~ 0)
    nz = np.abs(want) > 0
    strict = float((err[nz] / np.abs(want.astype(np.float64))[nz]).max()) if nz.any() else 0.0
    u = ulps(got, want)
    print(f"mel parity: max strict rel {strict:.3g}, max {int(u.max())} ulp, "
          f"{100 * np.mean(u == 0):.1f}% bit-identical, {100 * np.mean(u <= 1):.2f}% within 1 ulp")
    assert strict < 1e-4, strict  # no cell needs the floor of 1 on these inputs
    return float(np.mean(got == want))


def test_golden_tone():
    blob = open(os.path.join(GOLDEN, "mel_golden.bin"), "rb").read()
    nf, nm = np.frombuffer(blob[:8], "<u4")
    want = np.frombuffer(blob[8:], "<f4").reshape(nf, nm)
    pcm = np.fromfile(os.path.join(GOLDEN, "tone440_1s.s16"), "<i2")
    mel = api.compute_mel(api.AudioBuffer(pcm))
    assert mel.n_frames == nf and mel.n_mels == nm
    exact = close(mel.data, want)
    assert exact > 0.5
    assert int(np.argmax(mel.data.sum(0))) == 11  # media_tests.cpp:99-117


def test_stock_clip_and_random(reference):
    pcm = np.fromfile(os.path.join(GOLDEN, "stock10s.s16"), "<i2")
    mel = api.compute_mel(api.AudioBuffer(pcm))
    assert mel.n_frames == 622
    close(mel.data, reference.compute_mel(pcm))
    rng = np.random.default_rng(7)
    for n in (1024, 1279, 1280, 4097, 33333):
        pcm = rng.integers(-32768, 32767, n, dtype=np.int16)
        close(api.compute_mel(api.AudioBuffer(pcm)).data, reference.compute_mel(pcm))


def test_short_and_silent():
    assert api.compute_mel(api.AudioBuffer(np.zeros(1023, np.int16))).n_frames == 0
    mel = api.compute_mel(api.AudioBuffer(np.zeros(4096, np.int16)))
    assert mel.n_frames == 13
    assert np.all(mel.data == np.float32(np.log(1e-10)))  # media_tests.cpp:119-126


@pytest.mark.parametrize("fft,hop,n_mels,fmax", [(512, 128, 40, 8000.0), (2048, 256, 80, 7600.0),
                                                 (1024, 160, 64, 4000.0),
                                                 # fast path, band schedules with 1-2 bin and
                                                 # empty bands (-> ln 1e-10) and a single band
                                                 (1024, 256, 512, 8000.0), (1024, 256, 1, 8000.0)])
def test_other_configs(reference, fft, hop, n_mels, fmax):
    cfg = api.MelConfig(16000, fft, hop, n_mels, 0.0, fmax)
    pcm = reference.render_pattern(Pattern(), 3000)
    got = api.compute_mel(api.AudioBuffer(pcm), cfg).data
    want = reference.compute_mel(pcm, fft=fft, hop=hop, n_mels=n_mels, fmax=fmax)
    close(got, want)


def test_config_errors():
    for bad in (api.MelConfig(fft_size=1000), api.MelConfig(hop=0), api.MelConfig(n_mels=0),
                api.MelConfig(fmin=9000.0), api.MelConfig(sample_rate=0)):
        with pytest.raises(api.InvalidArgument):
            api.mel_frame_count(5000, bad)


def test_batch_device_segments(reference):
    """Ragged segments of one device-resident stream in one launch equal
    per-segment compute_mel (orchestrator.cpp:152 called per segment)."""
    torch = pytest.importorskip("torch")
    from streams import config2_streams
    streams = config2_streams(reference.render_pattern, seconds=20)
    pcm = np.concatenate(streams)
    dev = torch.from_numpy(pcm).cuda()
    rng = np.random.default_rng(2)
    offs, lens = [], []
    base = 0
    for s in streams:
        pos = 0
        while pos < len(s):
            ln = int(rng.integers(500, 48000))
            ln = min(ln, len(s) - pos)
            offs.append(base + pos)
            lens.append(ln)
            pos += ln
        base += len(s)
    frames = [0 if n < 1024 else 1 + (n - 1024) // 256 for n in lens]
    rows = np.concatenate([[0], np.cumsum(frames)[:-1]]).tolist()
    out = torch.zeros(int(sum(frames)), 80, dtype=torch.float32, device="cuda")
    ext = api.MelExtractor(api.MelConfig(), max_frames=1 << 16)
    torch.cuda.synchronize()  # torch's fill/copy run on its own stream
    ext.batch_device(dev.data_ptr(), offs, lens, out.data_ptr(), rows)
    ext.ctx.sync()
    got = out.cpu().numpy()
    for o, n, r, f in zip(offs, lens, rows, frames):
        if f:
            close(got[r:r + f], reference.compute_mel(pcm[o:o + n]))
