"""Host-side mirror of the reference operator API over the C ABI.

Same names, argument meaning and error behaviour as lipstream's
``Segmenter`` (segmenter.hpp:76-111), ``VadConfig`` (vad.hpp:19-24),
``compute_mel`` / ``mel_frame_count`` (mel.hpp:33-39) and the lip-sync stage
(visual_mocks.hpp:17-43), so parity tests read like the reference's own
tests.  All compute runs in liblsg.so on the GPU; this module only moves
buffers and keeps the per-stream bookkeeping a RawSegment needs.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import (Cut, DevRef, InvalidArgument, LogicError, MelCfg, SegCfg, SegMetrics, lib)


class SegmenterMode(enum.IntEnum):
    Baseline = 0
    Semantic = 1


class PeakMode(enum.IntEnum):
    Decay = 0
    MaxHold = 1
    Absolute = 2


class CutCause(enum.IntEnum):
    Pause = 0
    Forced = 1
    Eos = 2


@dataclass
class AudioBuffer:
    """include/lipstream/audio.hpp:12-20."""
    samples: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int16))
    sample_rate: int = 16000
    start: int = 0

    def duration_ms(self) -> int:
        return int(round(1000.0 * len(self.samples) / self.sample_rate))

    def empty(self) -> bool:
        return len(self.samples) == 0


@dataclass
class VadConfig:
    peak_mode: PeakMode = PeakMode.Decay
    peak_half_life_ms: float = 10000.0
    speech_threshold_db: float = -40.0
    frame_ms: int = 20


@dataclass
class SegmenterConfig:
    mode: SegmenterMode = SegmenterMode.Semantic
    vad: VadConfig = field(default_factory=VadConfig)
    min_silence_ms: int = 500
    min_segment_ms: int = 1500
    max_segment_ms: int = 10000
    sample_rate: int = 16000

    def to_c(self, flags_only: bool = False) -> SegCfg:
        return SegCfg(int(self.mode), int(self.vad.peak_mode), float(self.vad.peak_half_life_ms),
                      float(self.vad.speech_threshold_db), int(self.vad.frame_ms), int(self.min_silence_ms),
                      int(self.min_segment_ms), int(self.max_segment_ms), int(self.sample_rate),
                      1 if flags_only else 0)


@dataclass
class RawSegment:
    begin: int = 0
    end: int = 0
    audio: AudioBuffer = field(default_factory=AudioBuffer)
    confidence: float = 1.0
    cause: CutCause = CutCause.Eos

    def duration_ms(self) -> int:
        return self.end - self.begin


@dataclass
class BoundaryContext:
    pause_start: int
    silence_run_ms: int
    segment_span_ms: int


@dataclass
class BoundaryDecision:
    cut: bool = True
    confidence: float = 1.0
    cost_ms: float = 0.0


@dataclass
class SegmenterMetrics:
    frames: int = 0
    speech_frames: int = 0
    cuts_pause: int = 0
    cuts_forced: int = 0
    cuts_eos: int = 0
    scorer_calls: int = 0
    scorer_cost_ms: float = 0.0


class Context:
    """One GPU: device + stream (lsg_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = lib()
        h = C.c_void_p()
        self.lib.call("lsg_ctx_create", device, C.byref(h))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.lsg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self.lib.call("lsg_ctx_sync", self.h)

    def launches(self) -> int:
        n = C.c_int64()
        self.lib.call("lsg_ctx_launch_count", self.h, C.byref(n))
        return n.value

    def stream_ptr(self) -> int:
        p = C.c_void_p()
        self.lib.call("lsg_ctx_get_stream", self.h, C.byref(p))
        return p.value or 0

    def set_stream(self, ptr: int | None):
        """None: the context's own stream.  An int is a cudaStream_t; 0 (the
        legacy default stream, e.g. torch's default stream) maps to
        cudaStreamLegacy because NULL means "own stream" in the C ABI."""
        if ptr is None:
            self.lib.call("lsg_ctx_set_stream", self.h, C.c_void_p(0))
        else:
            self.lib.call("lsg_ctx_set_stream", self.h, C.c_void_p(ptr if ptr else 1))


_DEFAULT_CTX: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _DEFAULT_CTX:
        _DEFAULT_CTX[device] = Context(device)
    return _DEFAULT_CTX[device]


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class MultiStreamSegmenter:
    """n independent reference Segmenters on one GPU (lsg_seg)."""

    def __init__(self, cfg: SegmenterConfig, n_streams: int, max_push_samples: int, ctx: Context | None = None,
                 flags_only: bool = False):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.cfg = cfg
        self.n = n_streams
        h = C.c_void_p()
        c = cfg.to_c(flags_only)
        self.lib.call("lsg_seg_create", self.ctx.h, C.byref(c), n_streams, max_push_samples, C.byref(h))
        self.h = h

    def close(self):
        if self.h:
            self.lib.lsg_seg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def push_args(self, streams, chunks, starts, sample_rate=None):
        """Prebuilt lsg_seg_push arguments for device-resident chunks
        ((ptr, n) pairs): time the C-ABI call, not the ctypes marshalling."""
        n = len(streams)
        ids = (C.c_int32 * max(n, 1))(*streams)
        ptrs = (C.c_void_p * max(n, 1))(*[p for p, _ in chunks])
        lens = (C.c_int64 * max(n, 1))(*[ln for _, ln in chunks])
        st = (C.c_int64 * max(n, 1))(*starts)
        rate = self.cfg.sample_rate if sample_rate is None else sample_rate
        return (self.h, n, ids, ptrs, lens, st, rate, 1), (self.h, n, ids)

    def push_finish_prepared(self, args):
        """lsg_seg_push + lsg_seg_finish with push_args()'s arguments."""
        push, fin = args
        self.lib.call("lsg_seg_push", *push)
        self.lib.call("lsg_seg_finish", *fin)

    def push(self, streams, chunks, starts, sample_rate=None, on_device=False):
        """chunks: list of int16 numpy arrays (host) or raw device pointers + lengths."""
        n = len(streams)
        ids = (C.c_int32 * max(n, 1))(*streams)
        if on_device:
            ptrs = (C.c_void_p * max(n, 1))(*[p for p, _ in chunks])
            lens = (C.c_int64 * max(n, 1))(*[ln for _, ln in chunks])
            keep = None
        else:
            keep = [np.ascontiguousarray(c, np.int16) for c in chunks]
            ptrs = (C.c_void_p * max(n, 1))(*[k.ctypes.data for k in keep])
            lens = (C.c_int64 * max(n, 1))(*[len(k) for k in keep])
        st = (C.c_int64 * max(n, 1))(*starts)
        rate = self.cfg.sample_rate if sample_rate is None else sample_rate
        self.lib.call("lsg_seg_push", self.h, n, ids, ptrs, lens, st, rate, 1 if on_device else 0)
        del keep

    def finish(self, streams):
        n = len(streams)
        ids = (C.c_int32 * max(n, 1))(*streams)
        self.lib.call("lsg_seg_finish", self.h, n, ids)

    def take_cuts(self, stream: int) -> list[Cut]:
        n = C.c_int64()
        self.lib.call("lsg_seg_take_cuts", self.h, stream, None, 0, C.byref(n))
        buf = (Cut * max(n.value, 1))()
        self.lib.call("lsg_seg_take_cuts", self.h, stream, buf, n.value, C.byref(n))
        return [buf[i] for i in range(n.value)]

    def take_all_cuts(self) -> list[Cut]:
        n = C.c_int64()
        self.lib.call("lsg_seg_take_all_cuts", self.h, None, 0, C.byref(n))
        buf = (Cut * max(n.value, 1))()
        self.lib.call("lsg_seg_take_all_cuts", self.h, buf, n.value, C.byref(n))
        return [buf[i] for i in range(n.value)]

    def take_flags(self, stream: int) -> np.ndarray:
        n = C.c_int64()
        self.lib.call("lsg_seg_take_flags", self.h, stream, None, 0, C.byref(n))
        out = np.zeros(max(n.value, 1), np.uint8)
        self.lib.call("lsg_seg_take_flags", self.h, stream, _ptr(out), n.value, C.byref(n))
        return out[: n.value]

    def metrics(self, stream: int) -> SegmenterMetrics:
        m = SegMetrics()
        self.lib.call("lsg_seg_get_metrics", self.h, stream, C.byref(m))
        return SegmenterMetrics(m.frames, m.speech_frames, m.cuts_pause, m.cuts_forced, m.cuts_eos,
                                m.scorer_calls, m.scorer_cost_ms)


class Segmenter:
    """Drop-in for lipstream::Segmenter (segmenter.hpp:76-111).

    VAD, frame decisions and (without a scorer) the whole state machine run
    on the GPU.  With a BoundaryScorer the device returns per-frame speech
    flags and the state machine runs here, so scorer calls happen once per
    qualifying pause, in order, exactly as segmenter.cpp:84-90."""

    def __init__(self, cfg: SegmenterConfig | None = None, scorer=None, ctx: Context | None = None,
                 max_push_samples: int = 1 << 22):
        self.cfg = cfg or SegmenterConfig()
        self.scorer = scorer
        self._dev = MultiStreamSegmenter(self.cfg, 1, max_push_samples, ctx, flags_only=scorer is not None)
        self._rate = self.cfg.sample_rate
        self._pending = np.zeros(0, np.int16)  # samples of the open segment (host copy for RawSegment.audio)
        self._stage = 0
        self._finished = False
        self._metrics = SegmenterMetrics()
        # host state machine (scorer path only)
        self._fs = self.cfg.sample_rate * self.cfg.vad.frame_ms // 1000
        self._sm = dict(base=0, seg_start=0, consumed=0, speech_seen=False, silence_run=0, cand_open=False,
                        cand_cut=False, conf=1.0, pause_start=0, emitted=0)
        self._started = False

    def push(self, chunk: AudioBuffer) -> list[RawSegment]:
        samples = np.ascontiguousarray(chunk.samples, np.int16)
        # discipline checks happen in the C ABI (LogicError / InvalidArgument)
        self._dev.push([0], [samples], [int(chunk.start)], sample_rate=chunk.sample_rate)
        if len(samples) == 0:
            return []
        self._pending = np.concatenate([self._pending, samples])
        if not self._started:
            self._started = True
            self._sm["base"] = self._sm["seg_start"] = int(chunk.start)
        if self.scorer is None:
            return self._materialise(self._dev.take_cuts(0))
        return self._host_machine(self._dev.take_flags(0))

    def finish(self) -> list[RawSegment]:
        self._dev.finish([0])
        self._finished = True
        if self.scorer is None:
            return self._materialise(self._dev.take_cuts(0))
        # finish() (segmenter.cpp:120-145) on the host state
        sm = self._sm
        fs = self._fs
        stage = sm["emitted"] + len(self._pending) - sm["consumed"] * fs  # samples never framed
        tail_ms = stage * 1000 // self._rate
        if not sm["speech_seen"] or len(self._pending) == 0:
            self._pending = self._pending[:0]
            return []
        end = sm["base"] + sm["consumed"] * self.cfg.vad.frame_ms + tail_ms
        seg = RawSegment(sm["seg_start"], end, AudioBuffer(self._pending.copy(), self._rate, sm["seg_start"]),
                         1.0, CutCause.Eos)
        self._pending = self._pending[:0]
        self._metrics.cuts_eos += 1
        return [seg]

    def metrics(self) -> SegmenterMetrics:
        if self.scorer is None:
            return self._dev.metrics(0)
        m = self._dev.metrics(0)
        self._metrics.frames = m.frames
        self._metrics.speech_frames = m.speech_frames
        return self._metrics

    # -- helpers -------------------------------------------------------
    def _materialise(self, cuts) -> list[RawSegment]:
        out = []
        for c in cuts:
            k = int(c.sample_len)
            audio = AudioBuffer(self._pending[:k].copy(), self._rate, int(c.begin))
            self._pending = self._pending[k:]
            out.append(RawSegment(int(c.begin), int(c.end), audio, float(c.confidence), CutCause(c.cause)))
        return out

    def _emit(self, out, cut_ms, conf, cause):
        sm = self._sm
        split = (cut_ms - sm["seg_start"]) * self._rate // 1000
        audio = AudioBuffer(self._pending[:split].copy(), self._rate, sm["seg_start"])
        self._pending = self._pending[split:]
        out.append(RawSegment(sm["seg_start"], cut_ms, audio, conf, cause))
        sm["emitted"] += split
        sm["seg_start"] = cut_ms
        sm["speech_seen"] = False

    def _host_machine(self, flags) -> list[RawSegment]:
        """process_frame (segmenter.cpp:51-99) over device VAD decisions."""
        cfg, sm, out = self.cfg, self._sm, []
        fm = cfg.vad.frame_ms
        for sp in flags:
            f0 = sm["base"] + sm["consumed"] * fm
            f1 = f0 + fm
            if sp:
                if sm["speech_seen"] and sm["silence_run"] >= cfg.min_silence_ms and sm["cand_open"] and sm["cand_cut"]:
                    self._emit(out, sm["pause_start"] + sm["silence_run"] // 2, sm["conf"], CutCause.Pause)
                    self._metrics.cuts_pause += 1
                sm["silence_run"] = 0
                sm["cand_open"] = False
                sm["cand_cut"] = False
                sm["speech_seen"] = True
            else:
                if sm["silence_run"] == 0:
                    sm["pause_start"] = f0
                sm["silence_run"] += fm
                if not sm["cand_open"] and sm["silence_run"] >= cfg.min_silence_ms and sm["speech_seen"]:
                    sm["cand_open"] = True
                    sm["cand_cut"] = True
                    sm["conf"] = 1.0
                    if cfg.mode == SegmenterMode.Semantic:
                        if sm["pause_start"] - sm["seg_start"] < cfg.min_segment_ms:
                            sm["cand_cut"] = False
                        elif self.scorer is not None:
                            d = self.scorer(BoundaryContext(sm["pause_start"], sm["silence_run"],
                                                            sm["pause_start"] - sm["seg_start"]))
                            self._metrics.scorer_calls += 1
                            self._metrics.scorer_cost_ms += d.cost_ms
                            sm["cand_cut"] = bool(d.cut)
                            sm["conf"] = float(d.confidence)
            if cfg.mode == SegmenterMode.Semantic and sm["speech_seen"] and f1 - sm["seg_start"] >= cfg.max_segment_ms:
                self._emit(out, f1, 1.0, CutCause.Forced)
                self._metrics.cuts_forced += 1
            sm["consumed"] += 1
        return out


# --------------------------------------------------------------------- mel
@dataclass(frozen=True)
class MelConfig:
    """include/lipstream/mel.hpp:12-19."""
    sample_rate: int = 16000
    fft_size: int = 1024
    hop: int = 256
    n_mels: int = 80
    fmin: float = 0.0
    fmax: float = 8000.0

    def to_c(self) -> MelCfg:
        return MelCfg(self.sample_rate, self.fft_size, self.hop, self.n_mels, self.fmin, self.fmax)


@dataclass
class MelSpectrogram:
    n_frames: int = 0
    n_mels: int = 0
    data: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.float32))  # [frame][mel]

    def at(self, frame: int, mel: int) -> float:
        return float(self.data[frame, mel])


def mel_frame_count(n_samples: int, cfg: MelConfig = MelConfig()) -> int:
    c = cfg.to_c()
    f = C.c_int64()
    lib().call("lsg_mel_frames", n_samples, C.byref(c), C.byref(f))
    return f.value


class MelExtractor:
    """A reusable lsg_mel handle (tables built once)."""

    def __init__(self, cfg: MelConfig = MelConfig(), max_frames: int = 1 << 16, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.cfg = cfg
        c = cfg.to_c()
        h = C.c_void_p()
        self.lib.call("lsg_mel_create", self.ctx.h, C.byref(c), max_frames, C.byref(h))
        self.h = h
        self.max_frames = max_frames

    def close(self):
        if self.h:
            self.lib.lsg_mel_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __call__(self, audio: AudioBuffer) -> MelSpectrogram:
        pcm = np.ascontiguousarray(audio.samples, np.int16)
        F = mel_frame_count(len(pcm), self.cfg)
        out = np.zeros((max(F, 1), self.cfg.n_mels), np.float32)
        f = C.c_int64()
        self.lib.call("lsg_mel_compute", self.h, _ptr(pcm), len(pcm), _ptr(out), C.byref(f))
        return MelSpectrogram(f.value, self.cfg.n_mels, out[: f.value])

    def batch_device(self, pcm_dev: int, offsets, lengths, out_dev: int, out_rows):
        n = len(offsets)
        o = (C.c_int64 * max(n, 1))(*offsets)
        ln = (C.c_int64 * max(n, 1))(*lengths)
        r = (C.c_int64 * max(n, 1))(*out_rows)
        self.lib.call("lsg_mel_compute_batch", self.h, n, C.c_void_p(pcm_dev), o, ln, C.c_void_p(out_dev), r)


_MEL_CACHE: dict = {}


def compute_mel(audio: AudioBuffer, cfg: MelConfig = MelConfig()) -> MelSpectrogram:
    """Drop-in for compute_mel (mel.hpp:39)."""
    F = mel_frame_count(len(audio.samples), cfg)  # validates like mel.cpp:27-37
    key = cfg
    ext = _MEL_CACHE.get(key)
    if ext is None or ext.max_frames < F:
        ext = MelExtractor(cfg, max(F, 1 << 12))
        _MEL_CACHE[key] = ext
    return ext(audio)


def fft_radix2(buf: np.ndarray) -> None:
    """Drop-in for fft_radix2 (mel.hpp:42, mel.cpp:46-70): in-place radix-2
    FFT of a complex128 array on the GPU, bit-identical to the reference;
    InvalidArgument unless len(buf) is a power of two (<= 8192)."""
    if buf.dtype != np.complex128 or not buf.flags.c_contiguous:
        raise TypeError("fft_radix2: needs a C-contiguous complex128 array (std::vector<std::complex<double>>)")
    ctx = default_context()
    ctx.lib.call("lsg_fft_radix2", ctx.h, _ptr(buf), len(buf), 1)


def synth_pattern(lead_silence_ms: int, bursts, tone_hz: float, amplitude: float, total_ms: int,
                  sample_rate: int = 16000) -> np.ndarray:
    """render_pattern restated in liblsg (workload generation)."""
    n = C.c_int64()
    sp = (C.c_int64 * len(bursts))(*[b[0] for b in bursts])
    pa = (C.c_int64 * len(bursts))(*[b[1] for b in bursts])
    cap = total_ms * sample_rate // 1000
    out = np.zeros(max(cap, 1), np.int16)
    lib().call("lsg_synth_pattern", lead_silence_ms, len(bursts), sp, pa, tone_hz, amplitude, total_ms, sample_rate,
               _ptr(out), cap, C.byref(n))
    return out[: n.value]


__all__ = ["AudioBuffer", "BoundaryContext", "BoundaryDecision", "Context", "CutCause", "InvalidArgument",
           "LogicError", "MelConfig", "MelExtractor", "MelSpectrogram", "MultiStreamSegmenter", "PeakMode",
           "RawSegment", "Segmenter", "SegmenterConfig", "SegmenterMetrics", "SegmenterMode", "VadConfig",
           "compute_mel", "default_context", "mel_frame_count", "synth_pattern"]


# ------------------------------------------------------------ A/V alignment
@dataclass
class AlignResult:
    """align.hpp:17-21."""
    offset_ms: int = 0  # positive: motion lags the audio
    peak_corr: float = 0.0
    low_confidence: bool = False


class AlignRes(C.Structure):
    _fields_ = [("offset_ms", C.c_int64), ("peak_corr", C.c_double), ("low_confidence", C.c_int32),
                ("pad", C.c_int32)]


class _DevArrays:
    """Device copies of host arrays (the drop-ins take host data, like the
    reference's const references)."""

    def __init__(self, ctx: Context, *arrays):
        self.ctx, self.ptrs = ctx, []
        for a in arrays:
            p = C.c_void_p()
            ctx.lib.call("lsg_dev_alloc", ctx.h, max(a.nbytes, 16), C.byref(p))
            if a.nbytes:
                ctx.lib.call("lsg_copy", ctx.h, p, _ptr(a), a.nbytes)
            self.ptrs.append(p)

    def free(self):
        for p in self.ptrs:
            self.ctx.lib.lsg_dev_free(self.ctx.h, p)
        self.ptrs = []


def _i64(xs):
    return (C.c_int64 * max(len(xs), 1))(*[int(x) for x in xs])


def energy_envelope_ms(audio: AudioBuffer, ctx: Context | None = None) -> np.ndarray:
    """Drop-in for energy_envelope_ms (align.hpp:12): RMS of 10 ms hops, held per ms (GPU)."""
    return energy_envelopes([audio], ctx)[0]


def energy_envelopes(audios, ctx: Context | None = None) -> list[np.ndarray]:
    """Batched energy_envelope_ms: one lsg_align_energy call for many buffers."""
    ctx = ctx or default_context()
    if not audios:
        return []
    rate = audios[0].sample_rate
    if any(a.sample_rate != rate for a in audios):
        raise ValueError("energy_envelopes: one sample rate per batch")
    pcm = [np.ascontiguousarray(a.samples, np.int16) for a in audios]
    offs = np.cumsum([0] + [len(p) for p in pcm[:-1]])
    lens = [int(round(1000.0 * len(p) / rate)) if rate > 0 else 0 for p in pcm]
    oo = np.cumsum([0] + lens[:-1])
    allpcm = np.concatenate(pcm) if sum(len(p) for p in pcm) else np.zeros(1, np.int16)
    out = np.zeros(max(sum(lens), 1), np.float64)
    dev = _DevArrays(ctx, allpcm, out)
    try:
        got = (C.c_int64 * len(pcm))()
        ctx.lib.call("lsg_align_energy", ctx.h, len(pcm), dev.ptrs[0], _i64(offs), _i64([len(p) for p in pcm]), rate,
                     dev.ptrs[1], _i64(oo), got)
        ctx.lib.call("lsg_copy", ctx.h, _ptr(out), dev.ptrs[1], out.nbytes)
        ctx.sync()
    finally:
        dev.free()
    return [out[o:o + n].copy() for o, n in zip(oo, lens)]


def motion_envelope_ms(frames, t0: int, span: int, ctx: Context | None = None) -> np.ndarray:
    """Drop-in for motion_envelope_ms (align.hpp:16): frames = [(ts, mouth_motion)] sorted by ts (GPU)."""
    if span < 0:
        raise ValueError("align: negative span")
    ctx = ctx or default_context()
    ts = np.ascontiguousarray([f[0] for f in frames] or [0], np.int64)
    mo = np.ascontiguousarray([f[1] for f in frames] or [0.0], np.float64)
    out = np.zeros(max(span, 1), np.float64)
    dev = _DevArrays(ctx, ts, mo, out)
    try:
        ctx.lib.call("lsg_align_motion", ctx.h, 1, dev.ptrs[0], dev.ptrs[1], _i64([0]), _i64([len(frames)]),
                     _i64([t0]), _i64([span]), dev.ptrs[2], _i64([0]))
        ctx.lib.call("lsg_copy", ctx.h, _ptr(out), dev.ptrs[2], out.nbytes)
        ctx.sync()
    finally:
        dev.free()
    return out[:span].copy()


def align_envelopes(energy, motion, max_lag: int = 50, ctx: Context | None = None) -> AlignResult:
    """Drop-in for align_envelopes (align.hpp:33-35) (GPU)."""
    return align_batch([(energy, motion)], max_lag, ctx)[0]


def align_batch(pairs, max_lag: int = 50, ctx: Context | None = None) -> list[AlignResult]:
    """align_envelopes for many (energy, motion) pairs in one lsg_align_batch call."""
    ctx = ctx or default_context()
    if not pairs:
        return []
    es = [np.ascontiguousarray(e, np.float64) for e, _ in pairs]
    ms = [np.ascontiguousarray(m, np.float64) for _, m in pairs]
    eo, mo = np.cumsum([0] + [len(e) for e in es[:-1]]), np.cumsum([0] + [len(m) for m in ms[:-1]])
    ea = np.concatenate(es) if sum(len(e) for e in es) else np.zeros(1)
    ma = np.concatenate(ms) if sum(len(m) for m in ms) else np.zeros(1)
    dev = _DevArrays(ctx, ea, ma)
    res = (AlignRes * len(pairs))()
    try:
        ctx.lib.call("lsg_align_batch", ctx.h, len(pairs), dev.ptrs[0], _i64(eo), _i64([len(e) for e in es]),
                     dev.ptrs[1], _i64(mo), _i64([len(m) for m in ms]), max_lag, res)
    finally:
        dev.free()
    return [AlignResult(int(r.offset_ms), float(r.peak_corr), bool(r.low_confidence)) for r in res]


# ------------------------------------------------------ face crops (f1)
@dataclass
class KalmanConfig:
    """kalman.hpp:8-12."""
    process_noise: float = 1e-2
    measurement_noise: float = 25.0
    initial_variance: float = 1e6


class KalmanCfg(C.Structure):
    _fields_ = [("process_noise", C.c_double), ("measurement_noise", C.c_double), ("initial_variance", C.c_double)]


def mock_face_detect(frame_index: int, seed: int) -> tuple:
    """visual_mocks.cpp:10-22 -> (cx, cy, w, h)."""
    b = np.zeros(4, np.float64)
    lib().call("lsg_face_mock_detect", int(frame_index), C.c_uint64(seed & ((1 << 64) - 1)), _ptr(b))
    return tuple(float(x) for x in b)


def track_faces(segments, seed: int = 0, cfg: KalmanConfig = KalmanConfig(), ctx: Context | None = None):
    """The detect + smooth loop of orchestrator.cpp:115-129 for many segments
    in one call.  segments: list of (ts[], frame_index[], faces or None),
    faces an [n, 4] array with NaN rows for frames without a box.  Returns
    per segment (boxes [n, 4], velocities [n, 2]); raises RuntimeError where
    KalmanBoxFilter would throw."""
    ctx = ctx or default_context()
    if not segments:
        return []
    lens = [len(s[0]) for s in segments]
    offs = np.cumsum([0] + lens[:-1])
    F = max(sum(lens), 1)
    ts = np.zeros(F, np.int64)
    fi = np.zeros(F, np.int64)
    has = np.zeros(F, np.int32)
    faces = np.zeros((F, 4), np.float64)
    for (t, f, fa), o, n in zip(segments, offs, lens):
        ts[o:o + n] = t
        fi[o:o + n] = f
        if fa is not None:
            fa = np.asarray(fa, np.float64).reshape(n, 4)
            ok = ~np.isnan(fa).all(axis=1)
            has[o:o + n] = ok
            faces[o:o + n] = np.where(ok[:, None], fa, 0.0)
    box = np.zeros((F, 4), np.float64)
    vel = np.zeros((F, 2), np.float64)
    dev = _DevArrays(ctx, ts, fi, has, faces, box, vel)
    st = (C.c_int32 * len(segments))()
    c = KalmanCfg(cfg.process_noise, cfg.measurement_noise, cfg.initial_variance)
    try:
        ctx.lib.call("lsg_face_track", ctx.h, len(segments), _i64(offs), _i64(lens), dev.ptrs[0], dev.ptrs[1],
                     dev.ptrs[2], dev.ptrs[3], C.c_uint64(seed & ((1 << 64) - 1)), C.byref(c), dev.ptrs[4],
                     dev.ptrs[5], st)
        ctx.lib.call("lsg_copy", ctx.h, _ptr(box), dev.ptrs[4], box.nbytes)
        ctx.lib.call("lsg_copy", ctx.h, _ptr(vel), dev.ptrs[5], vel.nbytes)
        ctx.sync()
    finally:
        dev.free()
    for i, s_ in enumerate(st):
        if s_:
            raise RuntimeError(f"kalman: segment {i} diverged or had a bad measurement / time step")
    return [(box[o:o + n].copy(), vel[o:o + n].copy()) for o, n in zip(offs, lens)]


def crop96(frames: np.ndarray, frame_of, boxes, ctx: Context | None = None) -> np.ndarray:
    """Bilinear 96x96 crops: frames [F, H, W, 3] u8, frame_of [n], boxes [n, 4] -> [n, 96, 96, 3] u8."""
    ctx = ctx or default_context()
    frames = np.ascontiguousarray(frames, np.uint8)
    fo = np.ascontiguousarray(frame_of, np.int64)
    bx = np.ascontiguousarray(boxes, np.float64).reshape(-1, 4)
    out = np.zeros((len(fo), 96, 96, 3), np.uint8)
    dev = _DevArrays(ctx, frames, fo, bx, out)
    try:
        ctx.lib.call("lsg_face_crop", ctx.h, len(fo), dev.ptrs[0], frames.shape[1], frames.shape[2], dev.ptrs[1],
                     dev.ptrs[2], dev.ptrs[3])
        ctx.lib.call("lsg_copy", ctx.h, _ptr(out), dev.ptrs[3], out.nbytes)
        ctx.sync()
    finally:
        dev.free()
    return out


# ------------------------------------------------ zero-copy stage hand-off
class DeviceRegistry:
    """Device buffers keyed by (segment uuid, kind) -- SURVEY.md §8 f3.
    Stages exchange `wire.Ref`s (48 bytes on the wire, wire.*_ref codecs)
    instead of the payload bytes the reference's codecs copy
    (stage.cpp:176-301).  Errors: duplicate key / stale reference ->
    LogicError; arena exhausted -> LsgError (ERUNTIME)."""

    def __init__(self, arena_bytes: int, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        h = C.c_void_p()
        self.lib.call("lsg_reg_create", self.ctx.h, int(arena_bytes), C.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.lsg_reg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _uuid(u) -> C.Array:
        b = bytes(u)
        if len(b) != 16:
            raise ValueError("uuid must be 16 bytes")
        return (C.c_uint8 * 16).from_buffer_copy(b)

    @staticmethod
    def _to_py(r: DevRef):
        from .wire import Ref
        return Ref(bytes(r.uuid), r.kind, r.device, r.generation, r.offset, r.bytes)

    @staticmethod
    def _to_c(ref) -> DevRef:
        r = DevRef()
        C.memmove(r.uuid, bytes(ref.uuid), 16)
        r.kind, r.device, r.generation, r.offset, r.bytes = ref.kind, ref.device, ref.generation, ref.offset, ref.bytes
        return r

    def put(self, uuid, kind: int, src, nbytes: int | None = None):
        """Copy a host array / device pointer into the arena (async on the
        context stream); returns the Ref."""
        if isinstance(src, np.ndarray):
            src = np.ascontiguousarray(src)
            ptr, n = src.ctypes.data, src.nbytes if nbytes is None else nbytes
            keep = src
        else:
            ptr, n, keep = int(src), int(nbytes), None
        r = DevRef()
        self.lib.call("lsg_reg_put", self.h, self._uuid(uuid), kind, C.c_void_p(ptr), n, C.byref(r))
        if keep is not None:  # host source: the async copy must finish before the array may go
            self.ctx.sync()
        return self._to_py(r)

    def put_view(self, uuid, kind: int, dev_ptr: int, nbytes: int):
        """Adopt a caller-owned device range (no copy)."""
        r = DevRef()
        self.lib.call("lsg_reg_put_view", self.h, self._uuid(uuid), kind, C.c_void_p(dev_ptr), int(nbytes), C.byref(r))
        return self._to_py(r)

    def alloc(self, uuid, kind: int, nbytes: int):
        """Arena space for a producer to write into: (device pointer, Ref)."""
        r, p = DevRef(), C.c_void_p()
        self.lib.call("lsg_reg_alloc", self.h, self._uuid(uuid), kind, int(nbytes), C.byref(p), C.byref(r))
        return p.value or 0, self._to_py(r)

    def resolve(self, ref) -> tuple[int, int]:
        p, n = C.c_void_p(), C.c_int64()
        self.lib.call("lsg_reg_resolve", self.h, C.byref(self._to_c(ref)), C.byref(p), C.byref(n))
        return p.value or 0, n.value

    def find(self, uuid, kind: int):
        r = DevRef()
        self.lib.call("lsg_reg_find", self.h, self._uuid(uuid), kind, C.byref(r))
        return self._to_py(r)

    def retain(self, ref):
        self.lib.call("lsg_reg_retain", self.h, C.byref(self._to_c(ref)))

    def release(self, ref):
        self.lib.call("lsg_reg_release", self.h, C.byref(self._to_c(ref)))

    def read(self, ref) -> bytes:
        """D2H copy of a buffer (for consumers that really need host bytes)."""
        p, n = self.resolve(ref)
        out = np.empty(n, np.uint8)
        if n:
            self.lib.call("lsg_copy", self.ctx.h, C.c_void_p(out.ctypes.data), C.c_void_p(p), n)
            self.ctx.sync()
        return out.tobytes()

    def stats(self) -> dict:
        u, e, pk = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib.call("lsg_reg_stats", self.h, C.byref(u), C.byref(e), C.byref(pk))
        return {"used": u.value, "entries": e.value, "peak": pk.value}


def devref_encode(ref) -> bytes:
    """lsg_devref_encode through the library (the wire.Ref.to_bytes layout)."""
    out = (C.c_uint8 * 48)()
    lib().call("lsg_devref_encode", C.byref(DeviceRegistry._to_c(ref)), out)
    return bytes(out)


def devref_decode(b: bytes):
    r = DevRef()
    buf = (C.c_uint8 * 48).from_buffer_copy(bytes(b))
    lib().call("lsg_devref_decode", buf, C.byref(r))
    return DeviceRegistry._to_py(r)
