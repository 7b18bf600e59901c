"""A/V alignment: energy_envelope_ms,
motion_envelope_ms and align_envelopes (align.cpp) -- the reference's own
cases (media_tests.cpp:294-378, acceptance_main.cpp:607-668).

CPU: the plain-C restatement (oracle) bit-identical to the reference build.
GPU: the library (lsg_align_*) bit-identical to the restatement, one call
for a whole batch of pairs."""
import numpy as np
import pytest

from _oracle import Pattern, splitmix64


def _shifted(energy, shift):
    """motion lagging the audio by `shift` ms (media_tests.cpp:298-304)."""
    m = np.zeros_like(energy)
    for t in range(len(m)):
        src = t - shift
        if 0 <= src < len(energy):
            m[t] = energy[src]
    return m


def _random_pairs(reference, seed=808, trials=20):
    """media_tests.cpp:313-321: n in [400, 1000), u64_to_unit values."""
    st = [seed]
    pairs = []
    for _ in range(trials):
        n = 400 + splitmix64(st) % 600
        a = np.array([reference.u64_to_unit(splitmix64(st)) for _ in range(2 * n)])
        pairs.append((a[0::2].copy(), a[1::2].copy()))
    return pairs


def _brute(a, b, max_lag=50):
    """The tests' brute-force scan (media_tests.cpp:322-350)."""
    best, best_lag = -2.0, 0
    n = len(a)
    for lag in range(-max_lag, max_lag + 1):
        x = a[max_lag:n - max_lag]
        y = b[max_lag + lag:n - max_lag + lag]
        cnt = len(x)
        cov = (x * y).sum() / cnt - (x.sum() / cnt) * (y.sum() / cnt)
        va = (x * x).sum() / cnt - (x.sum() / cnt) ** 2
        vb = (y * y).sum() / cnt - (y.sum() / cnt) ** 2
        corr = cov / np.sqrt(va * vb)
        better = corr > best + 1e-12
        tie = abs(corr - best) <= 1e-12
        if better or (tie and (abs(lag) < abs(best_lag) or (abs(lag) == abs(best_lag) and lag < best_lag))):
            best, best_lag = corr, lag
    return best_lag, best


def test_energy_envelope_restated_vs_reference(reference, restated):
    pcm = reference.render_pattern(Pattern(), 3000)
    e_ref = reference.energy_envelope(pcm)
    assert len(e_ref) == 3000
    np.testing.assert_array_equal(restated.energy_envelope(pcm), e_ref)
    odd = pcm[:16000 * 2 + 77]  # partial last hop, rounding of the ms count
    np.testing.assert_array_equal(restated.energy_envelope(odd), reference.energy_envelope(odd))
    assert len(restated.energy_envelope(np.zeros(0, np.int16))) == 0


def test_shift_recovery_restated_vs_reference(reference, restated):
    energy = reference.energy_envelope(reference.render_pattern(Pattern(), 3000))
    for shift in range(-50, 51, 5):
        m = _shifted(energy, shift)
        got = restated.align(energy, m)
        assert got == reference.align(energy, m)
        assert got[0] == shift and not got[2] and got[1] > 0.99


def test_random_pairs_restated_vs_reference(reference, restated):
    for a, b in _random_pairs(reference):
        got = restated.align(a, b)
        assert got == reference.align(a, b)
        lag, corr = _brute(a, b)
        assert got[0] == lag and abs(got[1] - corr) < 1e-9


def test_flat_and_short_and_motion(reference, restated):
    flat, other = np.full(500, 0.25), np.arange(500) % 7.0
    assert restated.align(flat, other) == reference.align(flat, other) == (0, 0.0, True)
    assert restated.align(np.ones(100), np.ones(100)) == reference.align(np.ones(100), np.ones(100))
    frames = [(100, 1.0), (150, 0.5)]
    env = restated.motion_envelope(frames, 80, 100)  # media_tests.cpp:366-378
    np.testing.assert_array_equal(env, reference.motion_envelope(frames, 80, 100))
    assert env[0] == 0.0 and env[19] == 0.0 and env[20] == 1.0 and env[69] == 1.0 and env[70] == 0.5


# --------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_gpu_energy_and_motion_bit_exact(restated, reference):
    from paper_2512_18318_b200 import api
    pats = [Pattern(), Pattern(lead_silence_ms=0, bursts=[(900, 520)], tone_hz=311.0, amplitude=0.7)]
    pcms = [reference.render_pattern(p, ms) for p, ms in zip(pats, (3000, 10000))]
    pcms.append(pcms[0][:16000 * 2 + 77])
    pcms.append(np.zeros(0, np.int16))
    got = api.energy_envelopes([api.AudioBuffer(samples=p) for p in pcms])
    for g, p in zip(got, pcms):
        np.testing.assert_array_equal(g, restated.energy_envelope(p))
    frames = [(100, 1.0), (150, 0.5), (150, 0.25), (400, 2.0)]
    for t0, span in ((80, 100), (0, 600), (200, 0), (500, 50)):
        np.testing.assert_array_equal(api.motion_envelope_ms(frames, t0, span),
                                      restated.motion_envelope(frames, t0, span))
    with pytest.raises(ValueError):
        api.motion_envelope_ms(frames, 0, -1)


@pytest.mark.gpu
def test_gpu_align_batch_bit_exact(restated, reference):
    from paper_2512_18318_b200 import api
    energy = reference.energy_envelope(reference.render_pattern(Pattern(), 3000))
    pairs = [(energy, _shifted(energy, s)) for s in range(-50, 51, 5)]
    pairs += _random_pairs(reference)
    pairs += [(np.full(500, 0.25), np.arange(500) % 7.0), (np.ones(80), np.ones(80)), (energy[:90], energy[:100])]
    got = api.align_batch(pairs, 50)
    for (e, m), r in zip(pairs, got):
        want = restated.align(e, m)
        assert (r.offset_ms, r.peak_corr, r.low_confidence) == want
    for lag in (0, 7, 120):
        a, b = pairs[21]
        r = api.align_envelopes(a, b, lag)
        assert (r.offset_ms, r.peak_corr, r.low_confidence) == restated.align(a, b, lag)
    from paper_2512_18318_b200._lib import InvalidArgument
    with pytest.raises(InvalidArgument):
        api.align_envelopes(energy, energy, -1)


@pytest.mark.gpu
@pytest.mark.parametrize("rate", [44100, 48000, 8000])
def test_gpu_energy_other_rates_bit_exact(reference, rate):
    """Hops of 441 (hop % 8 != 0), 480 and 80 samples: the energy kernel's
    staging for non-16 kHz rates, bit-identical to the reference build; a
    rate whose staging would exceed shared memory is rejected with EINVAL."""
    from paper_2512_18318_b200 import api
    rng = np.random.default_rng(rate)
    pcms = [(rng.normal(0, 3000, n)).astype(np.int16) for n in (rate * 3 + 123, rate // 2, 1000)]
    got = api.energy_envelopes([api.AudioBuffer(samples=p, sample_rate=rate) for p in pcms])
    for g, p in zip(got, pcms):
        np.testing.assert_array_equal(g, reference.energy_envelope(p, rate))
    from paper_2512_18318_b200._lib import InvalidArgument
    with pytest.raises(InvalidArgument, match="rate too high"):
        api.energy_envelopes([api.AudioBuffer(samples=pcms[0], sample_rate=192000)])
