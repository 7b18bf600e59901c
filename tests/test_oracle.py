"""Pin the checkers before trusting them (CPU only).

The C restatement (oracle/lsg_oracle.c) must agree exactly with the
reference's own sources compiled into oracle/_ref, on the reference's own
known-answer cases (proj/tests/segmenter_tests.cpp, media_tests.cpp,
acceptance_main.cpp criterion 5/6) and on the committed golden vectors.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from _oracle import Pattern, random_chunks, random_pattern, splitmix64

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MEL_GOLDEN_SHA = "a098a3b05644ed2a08bb54939304a38969fd90a6df2ae81ec230c83ba1c79107"


def ends(cuts):
    return [c["end"] for c in cuts]


def begins(cuts):
    return [c["begin"] for c in cuts]


def both(restated, reference, pcm, cfg=None, chunk_seed=0, scorer=None):
    a, ma, ra = reference.segment(pcm, cfg, chunk_seed=chunk_seed, scorer=scorer)
    chunks = random_chunks(len(pcm), chunk_seed) if chunk_seed else None
    b, mb, rb = restated.segment(pcm, cfg, chunks=chunks, scorer=scorer)
    assert ra == rb
    assert a == b, "restatement diverges from the reference"
    if ra == 0:
        assert ma == mb
    return a


def test_stock_pattern_begins(restated, reference):
    # segmenter_tests.cpp:140-151
    pcm = reference.render_pattern(Pattern(), 8000)
    whole = both(restated, reference, pcm)
    assert begins(whole) == [0, 2300, 4300, 6300]
    for seed in (11, 12, 13):
        assert begins(both(restated, reference, pcm, chunk_seed=seed)) == [0, 2300, 4300, 6300]


def test_short_pauses_never_cut(restated, reference):
    # segmenter_tests.cpp:153-163
    pcm = reference.render_pattern(Pattern(0, [(1000, 400)]), 6000)
    cuts = both(restated, reference, pcm)
    assert len(cuts) == 1 and cuts[0]["end"] == 6000 and cuts[0]["cause"] == 2


def test_forced_split_semantic_only(restated, reference):
    # segmenter_tests.cpp:165-182
    pcm = reference.render_pattern(Pattern(0, [(20000, 600)]), 12000)
    sem = both(restated, reference, pcm)
    assert ends(sem) == [10000, 12000] and sem[0]["cause"] == 1
    base = both(restated, reference, pcm, {"mode": 0})
    assert ends(base) == [12000]


def test_baseline_vs_semantic_fixture(restated, reference):
    # segmenter_tests.cpp:184-198
    pcm = reference.render_pattern(Pattern(600, [(800, 600)]), 5600)
    assert ends(both(restated, reference, pcm, {"mode": 0})) == [1700, 3100, 4500, 5600]
    assert ends(both(restated, reference, pcm, {"mode": 1})) == [3100, 5600]


def test_scorer_veto(restated, reference):
    # segmenter_tests.cpp:200-230
    def make():
        calls = [0]

        def score(user, pause_start, silence, span, cut, conf, cost):
            calls[0] += 1
            cut[0] = 0 if calls[0] == 1 else 1
            conf[0] = 0.0 if calls[0] == 1 else 0.7
            cost[0] = 1.5
        return score, calls
    pcm = reference.render_pattern(Pattern(0, [(1600, 600)]), 6000)
    s1, c1 = make()
    a, ma, _ = reference.segment(pcm, scorer=s1)
    s2, c2 = make()
    b, mb, _ = restated.segment(pcm, scorer=s2)
    assert a == b and ma == mb
    assert ends(a) == [4100, 6000] and a[0]["confidence"] == 0.7 and a[0]["cause"] == 0
    assert c1[0] == c2[0] == 2 and ma["scorer_calls"] == 2 and ma["scorer_cost_ms"] == 3.0


def test_silence_only(restated, reference):
    pcm = np.zeros(16000 * 3, np.int16)
    assert both(restated, reference, pcm) == []


def test_config_rejections(restated, reference):
    # segmenter_tests.cpp:258-269 -> std::invalid_argument (rc 1)
    pcm = np.zeros(320, np.int16)
    for bad in ({"min_sil": 0}, {"max_seg": 1500}, {"rate": 44100}):
        assert reference.segment(pcm, bad)[2] == 1
        assert restated.segment(pcm, bad)[2] == 1


def test_randomized_streams_conserve_and_match(restated, reference):
    # segmenter_tests.cpp:82-116 (seed 2024, chunked by state+1)
    state = [2024]
    checked = 0
    while checked < 100:
        p = random_pattern(state)
        clip = 2000 + 20 * (splitmix64(state) % 376)
        if clip <= p.lead_silence_ms + 100:
            continue
        pcm = reference.render_pattern(p, clip)
        cuts = both(restated, reference, pcm, chunk_seed=(state[0] + 1) & ((1 << 64) - 1))
        checked += 1
        assert cuts[0]["begin"] == 0 and cuts[-1]["end"] == clip
        assert sum(c["sample_len"] for c in cuts) == clip * 16
        for k in range(1, len(cuts)):
            assert cuts[k]["begin"] == cuts[k - 1]["end"]
        assert cuts[-1]["cause"] == 2


def test_closed_form_cut_points(restated, reference):
    # segmenter_tests.cpp:118-138 (seed 77)
    state = [77]
    for _ in range(100):
        p = random_pattern(state)
        clip = 0
        for _t in range(256):
            cand = 2000 + 20 * (splitmix64(state) % 376)
            if cand > p.lead_silence_ms + 100 and reference.ends_in_speech(p, cand):
                clip = cand
                break
        if clip == 0:
            continue
        want = reference.expected_durations(p, clip)
        cuts = both(restated, reference, reference.render_pattern(p, clip))
        assert [c["end"] - c["begin"] for c in cuts] == want


def test_vad_modes_near_threshold(restated, reference):
    """Amplitude sweeps across -40 dB in all three peak modes (vad.cpp:26-53)."""
    rng = np.random.default_rng(5)
    for mode in (0, 1, 2):
        amps = np.concatenate([np.full(20, 0.9), np.geomspace(0.02, 0.001, 400), np.zeros(30),
                               np.geomspace(0.001, 0.05, 200)])
        t = np.arange(320)
        frames = [np.round(a * 32767 * np.sin(2 * np.pi * (t + rng.integers(0, 32)) / 32.0)) for a in amps]
        pcm = np.concatenate(frames).astype(np.int16)
        cfg = {"peak_mode": mode, "half_life": 200.0}
        both(restated, reference, pcm, cfg)
        both(restated, reference, pcm, dict(cfg, mode=0), chunk_seed=99)


def test_mel_golden_regenerates(reference, tmp_path):
    # media_tests.cpp:172-179 / acceptance_main.cpp:590-598: pure_tone(440, 1000)
    pcm = reference.render_pattern(Pattern(0, [(1000, 0)], tone_hz=440.0), 1000)
    mel = reference.compute_mel(pcm)
    path = str(tmp_path / "now.mel")
    reference.write_mel(path, mel)
    blob = open(path, "rb").read()
    assert hashlib.sha256(blob).hexdigest() == MEL_GOLDEN_SHA
    assert blob == open(os.path.join(GOLDEN, "mel_golden.bin"), "rb").read()


def test_restated_mel_matches_golden(restated):
    blob = open(os.path.join(GOLDEN, "mel_golden.bin"), "rb").read()
    n_frames, n_mels = np.frombuffer(blob[:8], "<u4")
    want = np.frombuffer(blob[8:], "<f4").reshape(n_frames, n_mels)
    pcm = np.fromfile(os.path.join(GOLDEN, "tone440_1s.s16"), "<i2")
    got = restated.compute_mel(pcm)
    assert got.shape == want.shape and np.array_equal(got, want)
    # band placement (media_tests.cpp:99-117): 440 Hz lands in band 11
    assert int(np.argmax(got.sum(0))) == 11


def test_restated_mel_bit_exact_random(restated, reference):
    rng = np.random.default_rng(11)
    for n in (1023, 1024, 1279, 1280, 5000, 16000):
        pcm = rng.integers(-32768, 32767, n, dtype=np.int16)
        a = reference.compute_mel(pcm)
        b = restated.compute_mel(pcm)
        assert a.shape == b.shape and np.array_equal(a, b)


def test_stock_clip_golden(restated):
    meta = json.load(open(os.path.join(GOLDEN, "stock10s.json")))
    pcm = np.fromfile(os.path.join(GOLDEN, "stock10s.s16"), "<i2")
    assert hashlib.sha256(pcm.tobytes()).hexdigest() == meta["pcm_sha256"]
    cuts, _, _ = restated.segment(pcm)
    assert [[c["begin"], c["end"], c["cause"]] for c in cuts] == meta["cuts"]
    mel = restated.compute_mel(pcm)
    assert mel.shape[0] == 622
    assert hashlib.sha256(mel.astype("<f4").tobytes()).hexdigest() == meta["mel_sha256"]


def test_mel_frame_count(reference):
    # media_tests.cpp:83-97
    for n, want in ((0, 0), (1023, 0), (1024, 1), (1279, 1), (1280, 2), (160000, 622)):
        assert reference.mel_frame_count(n) == want


def test_fft_matches_dft(restated, reference):
    # media_tests.cpp:128-150
    rng = np.random.default_rng(555)
    z = rng.random(16) - 0.5 + 1j * (rng.random(16) - 0.5)
    want = np.fft.fft(z)
    assert np.max(np.abs(reference.fft(z) - want)) < 1e-9
    assert np.array_equal(restated.fft(z), reference.fft(z))
    with pytest.raises(ValueError):
        restated.fft(np.zeros(12, complex))
