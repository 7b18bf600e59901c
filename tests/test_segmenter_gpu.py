"""Segmenter parity on the GPU, through the C ABI: bit-exact cut lists,
cut causes, confidences, sample spans and metrics against the reference's
own Segmenter (oracle/_ref) on the reference's known-answer cases and
seeded random streams."""
import numpy as np
import pytest

from _oracle import Pattern, random_chunks, random_pattern, splitmix64
from streams import config2_streams, near_threshold_stream

pytestmark = pytest.mark.gpu

api = pytest.importorskip("paper_2512_18318_b200.api")


def gpu_segment(pcm, cfg=None, chunks=None, start_ms=0, scorer=None):
    c = cfg or {}
    scfg = api.SegmenterConfig(
        mode=api.SegmenterMode(c.get("mode", 1)),
        vad=api.VadConfig(api.PeakMode(c.get("peak_mode", 0)), c.get("half_life", 10000.0), c.get("thr", -40.0),
                          c.get("frame_ms", 20)),
        min_silence_ms=c.get("min_sil", 500), min_segment_ms=c.get("min_seg", 1500),
        max_segment_ms=c.get("max_seg", 10000), sample_rate=c.get("rate", 16000))
    seg = api.Segmenter(scfg, scorer=scorer, max_push_samples=max(len(pcm), 1))
    out = []
    rate = scfg.sample_rate
    if chunks is None:
        chunks = [len(pcm)]
    off = 0
    for ln in chunks:
        out += seg.push(api.AudioBuffer(pcm[off:off + ln], rate, start_ms + off * 1000 // rate))
        off += ln
    out += seg.finish()
    return out, seg.metrics()


def as_cuts(segs):
    res, off = [], 0
    for s in segs:
        assert s.audio.start == s.begin
        res.append(dict(begin=s.begin, end=s.end, confidence=s.confidence, cause=int(s.cause),
                        sample_off=off, sample_len=len(s.audio.samples)))
        off += len(s.audio.samples)
    return res


def check(reference, pcm, cfg=None, chunk_seed=0):
    want, wm, rc = reference.segment(pcm, cfg, chunk_seed=chunk_seed)
    assert rc == 0
    chunks = random_chunks(len(pcm), chunk_seed) if chunk_seed else None
    segs, m = gpu_segment(pcm, cfg, chunks)
    assert as_cuts(segs) == want
    # samples of every RawSegment are the stream's own samples
    off = 0
    for s in segs:
        assert np.array_equal(s.audio.samples, pcm[off:off + len(s.audio.samples)])
        off += len(s.audio.samples)
    for k in ("frames", "speech_frames", "cuts_pause", "cuts_forced", "cuts_eos"):
        assert getattr(m, k) == wm[k], k
    return want


def test_known_answers(reference):
    pcm = reference.render_pattern(Pattern(), 8000)
    assert [c["begin"] for c in check(reference, pcm)] == [0, 2300, 4300, 6300]
    for seed in (11, 12, 13):
        check(reference, pcm, chunk_seed=seed)
    c = check(reference, reference.render_pattern(Pattern(0, [(1000, 400)]), 6000))
    assert [x["end"] for x in c] == [6000]
    p12 = reference.render_pattern(Pattern(0, [(20000, 600)]), 12000)
    assert [x["end"] for x in check(reference, p12)] == [10000, 12000]
    assert [x["end"] for x in check(reference, p12, {"mode": 0})] == [12000]
    fx = reference.render_pattern(Pattern(600, [(800, 600)]), 5600)
    assert [x["end"] for x in check(reference, fx, {"mode": 0})] == [1700, 3100, 4500, 5600]
    assert [x["end"] for x in check(reference, fx, {"mode": 1})] == [3100, 5600]
    assert check(reference, np.zeros(48000, np.int16)) == []


def test_randomized_streams_chunked(reference):
    state = [2024]
    done = 0
    while done < 100:
        p = random_pattern(state)
        clip = 2000 + 20 * (splitmix64(state) % 376)
        if clip <= p.lead_silence_ms + 100:
            continue
        check(reference, reference.render_pattern(p, clip), chunk_seed=(state[0] + 1) & ((1 << 64) - 1))
        done += 1


def test_config2_streams_batched(reference):
    """8 x 60 s in ONE push per stream (all streams one launch) + finish."""
    streams = config2_streams(reference.render_pattern)
    n = len(streams)
    ms = api.MultiStreamSegmenter(api.SegmenterConfig(), n, len(streams[0]))
    ms.push(list(range(n)), streams, [0] * n)
    ms.finish(list(range(n)))
    for s, pcm in enumerate(streams):
        want, wm, _ = reference.segment(pcm)
        got = [dict(begin=c.begin, end=c.end, confidence=c.confidence, cause=c.cause, sample_off=c.sample_off,
                    sample_len=c.sample_len) for c in ms.take_cuts(s)]
        assert got == want, f"stream {s}"
        m = ms.metrics(s)
        assert (m.frames, m.speech_frames, m.cuts_pause, m.cuts_forced, m.cuts_eos) == \
            tuple(int(wm[k]) for k in ("frames", "speech_frames", "cuts_pause", "cuts_forced", "cuts_eos"))


def test_vad_decisions_bit_exact_all_modes(reference):
    """Per-frame speech flags (flags_only) against VadTracker::update,
    including frames that sit exactly on the -40 dB threshold."""
    pcm = near_threshold_stream(30)
    rng = np.random.default_rng(3)
    noisy = (rng.normal(0, 1, 16000 * 20) * np.repeat(np.geomspace(3000, 3, 1000), 320)).astype(np.int16)
    for data in (pcm, noisy):
        for mode in (0, 1, 2):
            for thr in (-40.0, -35.0, -52.5):
                cfg = dict(peak_mode=mode, thr=thr, half_life=10000.0 if mode else 700.0)
                want, _ = reference.vad_frames(data, cfg)
                scfg = api.SegmenterConfig(vad=api.VadConfig(api.PeakMode(mode), cfg["half_life"], thr, 20))
                ms = api.MultiStreamSegmenter(scfg, 1, len(data), flags_only=True)
                ms.push([0], [data], [0])
                got = ms.take_flags(0)
                assert np.array_equal(got, want), (mode, thr, np.flatnonzero(got != want)[:10])


def test_exact_threshold_frames_decide_like_glibc(reference):
    # frame A: one sample of 2500 (peak -> 2500), frame B: rms/peak == 0.01 -> exactly -40 dB
    a = np.zeros(320, np.int16)
    a[0] = 2500
    b = np.zeros(320, np.int16)
    b[:125] = 40
    pcm = np.concatenate([a, b, a, b, b] * 20)
    for mode in (0, 1):
        cfg = dict(peak_mode=mode)
        want, db = reference.vad_frames(pcm, cfg)
        scfg = api.SegmenterConfig(vad=api.VadConfig(api.PeakMode(mode)))
        ms = api.MultiStreamSegmenter(scfg, 1, len(pcm), flags_only=True)
        ms.push([0], [pcm], [0])
        assert np.array_equal(ms.take_flags(0), want)


def test_scorer_veto_on_host_machine(reference):
    pcm = reference.render_pattern(Pattern(0, [(1600, 600)]), 6000)
    calls = []

    def scorer(ctx):
        calls.append(ctx)
        assert ctx.silence_run_ms >= 500 and ctx.segment_span_ms >= 1500
        return api.BoundaryDecision(False, 0.0, 1.5) if len(calls) == 1 else api.BoundaryDecision(True, 0.7, 1.5)
    segs, m = gpu_segment(pcm, scorer=scorer)
    assert [s.end for s in segs] == [4100, 6000]
    assert segs[0].confidence == 0.7 and segs[0].cause == api.CutCause.Pause
    assert len(calls) == 2 and m.scorer_calls == 2 and m.scorer_cost_ms == 3.0


def test_stream_discipline_and_config_errors(reference):
    seg = api.Segmenter(api.SegmenterConfig())
    a = api.AudioBuffer(reference.render_pattern(Pattern(), 1000), 16000, 0)
    seg.push(a)
    with pytest.raises(api.InvalidArgument):
        seg.push(api.AudioBuffer(a.samples, 16000, 5000))
    with pytest.raises(api.InvalidArgument):
        seg.push(api.AudioBuffer(a.samples, 8000, 1000))
    seg.finish()
    with pytest.raises(api.LogicError):
        seg.push(a)
    with pytest.raises(api.LogicError):
        seg.finish()
    for bad in (dict(min_silence_ms=0), dict(max_segment_ms=1500), dict(sample_rate=44100)):
        with pytest.raises(api.InvalidArgument):
            api.Segmenter(api.SegmenterConfig(**bad))


def test_scaled_streams_properties_and_oracle(restated, reference):
    """64 streams x 60 s (full config-2 length, 8x the streams): exact
    agreement with the C restatement and the reference's tiling contract."""
    rng = np.random.default_rng(1)
    n = 64
    state = [99]
    streams = []
    for i in range(n):
        p = random_pattern(state)
        p.tone_hz = float(150 + (i * 37) % 250)
        streams.append(reference.render_pattern(p, 60000))
    ms = api.MultiStreamSegmenter(api.SegmenterConfig(), n, 60 * 16000)
    # two pushes per stream with a ragged split, like a live feed
    cuts1 = [int(x) for x in rng.integers(1, 60 * 16000 - 1, n)]
    ms.push(list(range(n)), [s[:c] for s, c in zip(streams, cuts1)], [0] * n)
    ms.push(list(range(n)), [s[c:] for s, c in zip(streams, cuts1)], [c * 1000 // 16000 for c in cuts1])
    ms.finish(list(range(n)))
    for s in range(n):
        got = [dict(begin=c.begin, end=c.end, confidence=c.confidence, cause=c.cause, sample_off=c.sample_off,
                    sample_len=c.sample_len) for c in ms.take_cuts(s)]
        want, _, _ = restated.segment(streams[s], chunks=[cuts1[s], len(streams[s]) - cuts1[s]])
        assert got == want
        if got:
            assert sum(c["sample_len"] for c in got) == sum(c["sample_len"] for c in want)
            for k in range(1, len(got)):
                assert got[k]["begin"] == got[k - 1]["end"]


def test_device_resident_long_pushes_time_sliced(reference):
    """Pushes of >= 1024 frames per stream from device memory take the
    time-sliced path (K1 of slice s+1 overlapping the peak chain and the
    machine of slice s, segmenter.cu launch_sliced): cuts and metrics stay
    bit-identical to the reference, in one push and in a push that follows a
    frame-aligned first push (the peak / machine state carries across)."""
    torch = pytest.importorskip("torch")
    streams = config2_streams(reference.render_pattern)
    state = [4242]
    for i in range(8):
        p = random_pattern(state)
        p.tone_hz = float(160 + 29 * i)
        streams.append(reference.render_pattern(p, 60000))
    n, L = len(streams), 60 * 16000
    dev = torch.from_numpy(np.stack([s[:L] for s in streams])).cuda()
    base = dev.data_ptr()
    for split in (0, 320 * 75):  # one push; 1.5 s then the rest (aligned: no carry)
        ms = api.MultiStreamSegmenter(api.SegmenterConfig(), n, L)
        if split:
            ms.push(list(range(n)), [(base + s * L * 2, split) for s in range(n)], [0] * n, on_device=True)
        ms.push(list(range(n)), [(base + (s * L + split) * 2, L - split) for s in range(n)],
                [split // 16] * n, on_device=True)
        torch.cuda.synchronize()
        ms.finish(list(range(n)))
        for s in range(n):
            want, wm, _ = reference.segment(streams[s][:L])
            got = [dict(begin=c.begin, end=c.end, confidence=c.confidence, cause=c.cause, sample_off=c.sample_off,
                        sample_len=c.sample_len) for c in ms.take_cuts(s)]
            assert got == want, (split, s)
            m = ms.metrics(s)
            assert (m.frames, m.speech_frames, m.cuts_pause, m.cuts_forced, m.cuts_eos) == \
                tuple(int(wm[k]) for k in ("frames", "speech_frames", "cuts_pause", "cuts_forced", "cuts_eos"))
