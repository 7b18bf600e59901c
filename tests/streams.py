"""Seeded synthetic streams for the segmenter/mel parity cases (config 2).

Streams 0-5 use random_scenario(i+1)'s speech pattern (scenario.cpp:110-170),
cycled out to 60 s.  Stream 6 is a 14 s burst followed by silence and
shorter bursts (forced splits, trailing-silence drop).
Stream 7 is integer-built tone material whose level walks across the
-40 dB gate (H1 guard band, exact-threshold frames included).
"""
import numpy as np

from _oracle import M64, Pattern, splitmix64


def mix_u64(h: int, v: int) -> int:
    """include/lipstream/rng.hpp:21-25."""
    h ^= (v + 0x9E3779B97F4A7C15 + ((h << 6) & M64) + (h >> 2)) & M64
    s = [h & M64]
    return splitmix64(s)


def random_scenario_pattern(seed: int) -> Pattern:
    state = [mix_u64(seed, 0x5CE7A510)]

    def pick(lo, hi, step):
        n = (hi - lo) // step + 1
        return lo + step * (splitmix64(state) % n)
    p = Pattern()
    p.lead_silence_ms = pick(0, 600, 20)
    p.tone_hz = float(pick(150, 400, 1))
    p.bursts = []
    for _ in range(pick(1, 4, 1)):
        s = pick(600, 2000, 20)
        q = pick(520, 960, 40)
        p.bursts.append((s, q))
    return p


def near_threshold_stream(seconds: int, seed: int = 7) -> np.ndarray:
    """Square-ish integer tone frames whose amplitude sweeps around the
    -40 dB point of the decaying peak, plus frames built to land exactly on
    the threshold (max 25*j, sum of squares 20*j^2 after a reset)."""
    rng = np.random.default_rng(seed)
    fs = 320
    frames = []
    n_frames = seconds * 50
    amp = 20000
    for f in range(n_frames):
        k = f % 400
        if k < 30:                       # loud burst resets the peak
            a = amp
        elif k < 330:                    # level walks from -30 dB to -50 dB
            a = int(amp * 10 ** (-(30 + 20 * (k - 30) / 300) / 20))
        else:
            a = 0
        x = np.zeros(fs, np.int64)
        if a > 0:
            x[0::2] = a
            x[1::2] = -a
            jitter = rng.integers(-1, 2, fs)
            x = x + jitter * (a > 4)
        frames.append(x)
    pcm = np.concatenate(frames)
    # exact-threshold frames: peak 2500 (=25*100) frame, then 320 samples with
    # sum of squares 20*100^2 = 200000 -> rms/peak == 0.01 exactly
    for j0 in range(5, n_frames - 2, 777):
        pcm[j0 * fs:(j0 + 1) * fs] = 0
        pcm[j0 * fs] = 2500
        q = np.zeros(fs, np.int64)
        q[:125] = 40                    # 125 * 1600 = 200000
        pcm[(j0 + 1) * fs:(j0 + 2) * fs] = q
    return np.clip(pcm, -32768, 32767).astype(np.int16)


def long_burst_pattern() -> Pattern:
    return Pattern(300, [(14000, 2200), (1200, 700), (800, 540)], tone_hz=300.0, amplitude=0.5)


def config2_streams(render, seconds: int = 60):
    """8 x `seconds` streams; `render(pattern, total_ms)` -> int16 PCM."""
    out = []
    for i in range(6):
        out.append(render(random_scenario_pattern(i + 1), seconds * 1000))
    out.append(render(long_burst_pattern(), seconds * 1000))
    out.append(near_threshold_stream(seconds))
    return out
